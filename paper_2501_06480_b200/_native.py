"""ctypes binding of libfwa.so (the C-ABI declared in include/fwa.h).

This is the only place Python touches native code. There is no fallback:
if the shared library is missing or cannot be loaded, every hot-path call
raises ``NativeLibraryError`` immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (
    CapacityError,
    ContextError,
    FlashwinError,
    InvalidRangeError,
    PartitionError,
    ShapeError,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
# FWA_LIB_PATH: load an alternative build of the same C-ABI (A/B timing of kernel variants)
LIB_PATH = os.environ.get("FWA_LIB_PATH") or os.path.join(_HERE, "_lib", "libfwa.so")

FWA_F32, FWA_F16, FWA_BF16 = 0, 1, 2
KERNEL_AUTO, KERNEL_GENERIC, KERNEL_TC = 0, 1, 2


class NativeLibraryError(FlashwinError, RuntimeError):
    """libfwa.so is missing or unusable; the CUDA path cannot run."""


class CudaError(FlashwinError, RuntimeError):
    """A CUDA launch or runtime call inside libfwa failed."""


_STATUS = {
    1: ShapeError,
    2: CapacityError,
    3: InvalidRangeError,
    4: ContextError,
    5: CudaError,
    6: PartitionError,
}


class FwaDesc(ctypes.Structure):
    _fields_ = [
        ("num_windows", ctypes.c_int64),
        ("heads", ctypes.c_int32),
        ("seq_len", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("scale", ctypes.c_float),
        ("chunks", ctypes.c_int32),
        ("mask_windows", ctypes.c_int32),
        ("kernel", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("add_table", ctypes.c_void_p),
    ]


class FwaFootprint(ctypes.Structure):
    _fields_ = [
        ("kernel_fwd", ctypes.c_int32),
        ("kernel_bwd", ctypes.c_int32),
        ("smem_bytes_fwd", ctypes.c_int64),
        ("smem_bytes_bwd", ctypes.c_int64),
        ("tmem_cols_fwd", ctypes.c_int32),
        ("tmem_cols_bwd", ctypes.c_int32),
        ("paper_peak_fwd", ctypes.c_int64),
        ("paper_peak_bwd", ctypes.c_int64),
        ("hbm_bytes_fwd", ctypes.c_int64),
        ("hbm_bytes_bwd", ctypes.c_int64),
    ]


class FwaWinDesc(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int64),
        ("height", ctypes.c_int32),
        ("width", ctypes.c_int32),
        ("channels", ctypes.c_int32),
        ("window", ctypes.c_int32),
        ("shift", ctypes.c_int32),
        ("elem_bytes", ctypes.c_int32),
    ]


_vp = ctypes.c_void_p
_SIGNATURES = {
    "fwa_fwd": (ctypes.c_int, [ctypes.POINTER(FwaDesc), _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                               ctypes.c_size_t, _vp]),
    "fwa_fwd_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(FwaDesc), ctypes.c_int,
                                                  ctypes.c_int]),
    "fwa_add_table_bytes": (ctypes.c_size_t, [ctypes.POINTER(FwaDesc), ctypes.c_int, ctypes.c_int]),
    "fwa_build_add_table": (ctypes.c_int, [ctypes.POINTER(FwaDesc), _vp, _vp, _vp, ctypes.c_size_t,
                                           _vp]),
    "fwa_bwd": (
        ctypes.c_int,
        [ctypes.POINTER(FwaDesc), _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
         ctypes.c_size_t, _vp],
    ),
    "fwa_fwd_qkv": (ctypes.c_int, [ctypes.POINTER(FwaDesc), _vp, _vp, _vp, _vp, _vp,
                                   ctypes.c_size_t, _vp]),
    "fwa_bwd_qkv": (
        ctypes.c_int,
        [ctypes.POINTER(FwaDesc), _vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp],
    ),
    "fwa_bwd_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(FwaDesc), ctypes.c_int,
                                                  ctypes.c_int, ctypes.c_int]),
    "fwa_footprint": (ctypes.c_int, [ctypes.POINTER(FwaDesc), ctypes.POINTER(FwaFootprint)]),
    "fwa_window_partition": (ctypes.c_int, [ctypes.POINTER(FwaWinDesc), _vp, _vp, _vp]),
    "fwa_window_reverse": (ctypes.c_int, [ctypes.POINTER(FwaWinDesc), _vp, _vp, _vp]),
    "fwa_bias_gather": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, _vp, _vp]),
    "fwa_bias_scatter": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, _vp, _vp]),
    "fwa_shift_mask": (
        ctypes.c_int,
        [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_float, _vp, _vp],
    ),
    "fwa_fill_uniform": (
        ctypes.c_int,
        [ctypes.c_uint64, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_int32, _vp,
         _vp],
    ),
    "fwa_last_error": (ctypes.c_char_p, []),
    "fwa_abi_version": (ctypes.c_int, []),
    "fwa_launch_count": (ctypes.c_int64, []),
    "fwa_device_info": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)]),
    "fwa_device_flags": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint32)]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load libfwa.so once; raise NativeLibraryError if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (make -C paper_2501_06480_b200/csrc). There is no CPU fallback."
            )
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (restype, argtypes) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = restype
            fn.argtypes = argtypes
        _lib = lib
        return lib


def check(status: int, prefix: str = "") -> None:
    if status == 0:
        return
    msg = load().fwa_last_error().decode(errors="replace")
    exc = _STATUS.get(status, FlashwinError)
    raise exc(f"{prefix}{msg}" if prefix else msg)


def last_error() -> str:
    return load().fwa_last_error().decode(errors="replace")


def launch_count() -> int:
    return int(load().fwa_launch_count())


def device_info() -> tuple[int, int]:
    sm = ctypes.c_int32(0)
    l2 = ctypes.c_int64(0)
    load().fwa_device_info(ctypes.byref(sm), ctypes.byref(l2))
    return int(sm.value), int(l2.value)


def device_flags() -> int:
    f = ctypes.c_uint32(0)
    check(load().fwa_device_flags(ctypes.byref(f)))
    return int(f.value)
