"""B200-native Flash Window Attention (arXiv 2501.06480).

Drop-in for the reference package ``flashwin``'s hot path
(pkg/src/flashwin/__init__.py:19-45): the same names and signatures for
``TileConfig``, ``flash_forward``, ``flash_backward``, ``batched_flash_forward``,
``FlashContext``, ``TrafficReport``, ``ScratchpadArena``, ``peak_sram_*``,
``WindowConfig``, ``window_partition``, ``window_reverse``, ``Rng``,
``fill_uniform`` and the error classes — computed by hand-written sm_100a
kernels in ``_lib/libfwa.so`` (C-ABI: include/fwa.h). No CPU fallback.

Extensions: ``batched_flash_backward``, the autograd ``window_attention``
(with Swin bias/mask), ``relative_position_bias`` and device helpers in ``ops``.
"""

from . import ops
from ._native import NativeLibraryError
from .api import (
    BatchedContexts,
    HostArray,
    batched_flash_backward,
    batched_flash_forward,
    flash_backward,
    flash_forward,
)
from .autograd import (
    RelativePositionBias,
    WindowAttentionFunction,
    WindowAttentionQKVFunction,
    partition_windows,
    relative_position_bias,
    reverse_windows,
    window_attention,
    window_attention_qkv,
)
from .errors import (
    CapacityError,
    ContextError,
    FlashwinError,
    InvalidRangeError,
    NumericsError,
    OracleError,
    PartitionError,
    ShapeError,
)
from .rng import Rng, fill_uniform
from .swin import SwinWindowAttention, TorchSwinWindowAttention
from .tiling import (
    DEFAULT_CAPACITY_BYTES,
    FlashContext,
    ScratchpadArena,
    TileConfig,
    TrafficReport,
    merge_reports,
    peak_sram_backward,
    peak_sram_forward,
    resolve_r,
)
from .windowing import WindowConfig, window_partition, window_reverse

__version__ = "0.1.0"

__all__ = [
    "BatchedContexts",
    "CapacityError",
    "ContextError",
    "DEFAULT_CAPACITY_BYTES",
    "FlashContext",
    "FlashwinError",
    "HostArray",
    "InvalidRangeError",
    "NativeLibraryError",
    "NumericsError",
    "OracleError",
    "PartitionError",
    "RelativePositionBias",
    "Rng",
    "ScratchpadArena",
    "ShapeError",
    "SwinWindowAttention",
    "TileConfig",
    "TorchSwinWindowAttention",
    "TrafficReport",
    "WindowAttentionFunction",
    "WindowAttentionQKVFunction",
    "WindowConfig",
    "batched_flash_backward",
    "batched_flash_forward",
    "fill_uniform",
    "flash_backward",
    "flash_forward",
    "merge_reports",
    "ops",
    "peak_sram_backward",
    "partition_windows",
    "peak_sram_forward",
    "relative_position_bias",
    "resolve_r",
    "reverse_windows",
    "window_attention",
    "window_attention_qkv",
    "window_partition",
    "window_reverse",
]
