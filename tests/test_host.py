"""CPU-only tests: host logic, C-ABI exports and validation (no kernel launches)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2501_06480_b200 as fw
from paper_2501_06480_b200 import _native as nat
from paper_2501_06480_b200.tiling import backward_report, forward_report, merge_reports

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    with open(os.path.join(ROOT, "include", "fwa.h")) as f:
        header = f.read()
    declared = set(re.findall(r"\b(fwa_[a-z_0-9]+)\s*\(", header))
    assert declared, "no declarations parsed"
    lib = nat.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(nat.EXPORTED_SYMBOLS)
    assert lib.fwa_abi_version() == 2


def test_tileconfig_matches_reference_rules(golden):
    assert fw.TileConfig(r=4).chunk_width(64) == 16
    assert fw.TileConfig(r=4).chunk_width(10) == 3
    assert fw.TileConfig(r=4).chunk_spans(10) == [(0, 3), (3, 6), (6, 9), (9, 10)]
    with pytest.raises(fw.InvalidRangeError):
        fw.TileConfig(r=0)
    with pytest.raises(fw.InvalidRangeError):
        fw.TileConfig(r=1, elem_bytes=2)
    with pytest.raises(fw.InvalidRangeError):
        fw.TileConfig(r=1, scale=-1.0)
    with pytest.raises(fw.ShapeError):
        fw.TileConfig(r=5).chunk_width(4)
    with pytest.raises(fw.ShapeError):
        fw.TileConfig(r=3).chunk_width(4)
    scalars, _ = golden
    for p in scalars["peaks"]:
        cfg = fw.TileConfig(r=p["r"], elem_bytes=p["elem_bytes"])
        assert fw.peak_sram_forward(p["L"], p["C"], cfg) == p["fwd"]
        assert fw.peak_sram_backward(p["L"], p["C"], cfg) == p["bwd"]


def test_reports_merge_like_reference(golden):
    scalars, _ = golden
    b = scalars["batched70"]
    reps = [forward_report(1, 64, 64, 24576) for _ in range(16)]
    m = merge_reports(reps)
    assert m.loads == b["loads"] and m.stores == b["stores"] and m.peak_sram_bytes == b["peak"]
    for case in scalars["grid"][:10]:
        L, C = case["L"], case["C"]
        br = backward_report(1, L, C, case["bwd_peak"])
        assert br.loads == case["bwd_loads"] and br.stores == case["bwd_stores"]


def test_capacity_and_shape_errors_raised_before_device_use():
    # No GPU here: these must fail in validation, never reach CUDA.
    q = np.zeros((1024, 32))
    with pytest.raises(fw.CapacityError, match="131072"):
        fw.flash_forward(q, q, q, fw.TileConfig(r=2), fw.ScratchpadArena())
    with pytest.raises(fw.ShapeError):
        fw.flash_forward(np.zeros((2, 4)), np.zeros((2, 4)), np.zeros((2, 6)),
                         fw.TileConfig(r=1), fw.ScratchpadArena())
    with pytest.raises(fw.ContextError):
        fw.flash_backward(None, np.zeros((2, 2)), fw.ScratchpadArena())
    q4 = np.zeros((2, 2, 64, 64))
    with pytest.raises(fw.CapacityError, match=r"slice \(b=0, head=0\)"):
        fw.batched_flash_forward(q4, q4, q4, fw.TileConfig(r=1), [fw.ScratchpadArena(1024)])
    with pytest.raises(fw.InvalidRangeError):
        fw.batched_flash_forward(q4, q4, q4, fw.TileConfig(r=1), [])
    with pytest.raises(fw.PartitionError):
        fw.WindowConfig(H=10, W=10, C=3, k=3)
    with pytest.raises(fw.ShapeError):
        fw.WindowConfig(H=0, W=4, C=1, k=2)


def _desc(**kw):
    base = dict(N=4, h=3, L=49, d=32, dtype=1, scale=1.0, chunks=2, mask_windows=0, kernel="auto")
    base.update(kw)
    return fw.ops.make_desc(base["N"], base["h"], base["L"], base["d"], base["dtype"],
                            base["scale"], base["chunks"], base["mask_windows"], base["kernel"])


@pytest.mark.parametrize("kw,status", [
    (dict(), 0),
    (dict(N=0), 1),
    (dict(L=0), 1),
    (dict(chunks=0), 3),
    (dict(chunks=33), 1),
    (dict(d=4, chunks=3), 1),   # ceil(4/3)=2 leaves an empty chunk
    (dict(scale=float("nan")), 3),
    (dict(scale=-1.0), 3),
    (dict(dtype=7), 3),
])
def test_c_abi_validation_codes(kw, status):
    lib = nat.load()
    fp = nat.FwaFootprint()
    d = _desc(**kw)
    assert lib.fwa_footprint(ctypes.byref(d), ctypes.byref(fp)) == status
    if status:
        assert lib.fwa_last_error()


def test_c_abi_rejects_null_pointers_without_launching():
    lib = nat.load()
    d = _desc()
    before = lib.fwa_launch_count()
    assert lib.fwa_fwd(ctypes.byref(d), None, None, None, None, None, None, None, 0, None) == 1
    assert lib.fwa_launch_count() == before


def test_shard_ranges_cover_batch_exactly():
    from paper_2501_06480_b200.shard import shard_images

    for B, G in [(128, 1), (128, 2), (128, 8), (7, 3), (1, 2)]:
        shards = [shard_images(B, 64, r, G) for r in range(G)]
        assert shards[0].image_begin == 0 and shards[-1].image_end == B
        for a, b in zip(shards, shards[1:]):
            assert a.image_end == b.image_begin
        assert sum(s.windows for s in shards) == B * 64
        assert all(s.window_begin % 64 == 0 for s in shards)  # mask index n % nW preserved


def test_poly_exp2_restatement_accuracy_and_clamp():
    """Python restatement of fwa_sm100.cuh ex2_poly: degree-3 2^f on [-0.5, 0.5] with the
    exponent added as an integer. Relative error <= 8e-5 (below 16-bit P rounding) and no
    NaN / sign wrap for very negative inputs (clamped at -125)."""
    import numpy as np

    def ex2_poly(x):
        x = np.maximum(np.asarray(x, np.float32), np.float32(-125.0))
        t = (x + np.float32(12582912.0)).astype(np.float32)
        j = (t - np.float32(12582912.0)).astype(np.float32)
        f = (x - j).astype(np.float32)
        p = np.float32(0.05508868396282196) * f + np.float32(0.24260404706001282)
        p = (p * f + np.float32(0.6932762265205383)).astype(np.float32)
        p = (p * f + np.float32(0.9999289512634277)).astype(np.float32)
        bits = p.view(np.int32) + (t.view(np.int32) << 23)
        return bits.astype(np.int32).view(np.float32)

    x = np.linspace(-30.0, 0.0, 100001, dtype=np.float32)
    rel = np.abs(ex2_poly(x) / np.exp2(x.astype(np.float64)) - 1.0)
    assert rel.max() < 8e-5
    y = ex2_poly(np.array([-126.5, -150.0, -1e30, -np.inf], np.float32))
    assert np.all(np.isfinite(y)) and np.all(y >= 0) and np.all(y < 1e-37)


class _DenseLike:
    """The reference DenseTensor's surface (tensor.py:26-71): shape, a read-only float64
    ``.array`` view and no ``__getitem__``; stands in when /root/reference is absent."""

    __slots__ = ("_a",)

    def __init__(self, shape, data):
        a = np.asarray(data, dtype=np.float64).reshape(-1).copy()
        a.setflags(write=False)
        self._a = a.reshape(tuple(shape))

    @property
    def shape(self):
        return self._a.shape

    @property
    def array(self):
        return self._a


def _dense_classes():
    classes = [_DenseLike]
    ref = "/root/reference/pkg/src"
    if os.path.isdir(ref):
        import sys

        sys.path.insert(0, ref)
        try:
            from flashwin.tensor import DenseTensor

            classes.append(DenseTensor)
        finally:
            sys.path.remove(ref)
    return classes


@pytest.mark.parametrize("dense", _dense_classes())
def test_batched_contexts_slice_dense_tensors(dense):
    # harness.py:543-550 indexes contexts[b][head] of DenseTensor inputs: must not need
    # DenseTensor.__getitem__ (it has none)
    rng = np.random.default_rng(0)
    arrs = [rng.standard_normal((3, 2, 5, 4)) for _ in range(3)]
    q, k, v = (dense(a.shape, a) for a in arrs)
    ctxs = fw.BatchedContexts(q, k, v, fw.TileConfig(r=1))
    assert len(ctxs) == 3 and len(ctxs[0]) == 2
    c = ctxs[2][1]
    for got, a in zip((c.q, c.k, c.v), arrs):
        assert hasattr(got, "array") and got.shape == (5, 4)
        assert np.array_equal(got.array, a[2, 1])
    assert c.bias is None and c.mask is None and c.mask_windows == 0
    assert [len(x) for x in ctxs[0:2]] == [2, 2]


def test_batched_contexts_carry_bias_and_mask_per_slice():
    import torch

    B, h, L, C, nW = 5, 3, 4, 2, 2
    q, k, v = (torch.randn(B, h, L, C) for _ in range(3))
    bias = torch.randn(h, L, L)
    mask = torch.randn(nW, L, L)
    ctxs = fw.BatchedContexts(q, k, v, fw.TileConfig(r=1), bias, mask)
    for b in range(B):
        for hd in range(h):
            c = ctxs[b][hd]
            assert torch.equal(c.q, q[b, hd]) and torch.equal(c.bias, bias[hd])
            assert torch.equal(c.mask, mask[b % nW]) and c.mask_windows == 1


def _desc_v2(N, h, L, d, dtype=1, mask_windows=0, kernel=0):
    return nat.FwaDesc(num_windows=N, heads=h, seq_len=L, head_dim=d, dtype=dtype, scale=0.2,
                       chunks=1, mask_windows=mask_windows, kernel=kernel, reserved=0,
                       add_table=None)


def test_workspace_queries_size_the_add_table_and_partials_exactly():
    # ABI 2: scratch is caller workspace; the library sizes it (no device work here)
    lib = nat.load()
    q = lambda f, *a: int(getattr(lib, f)(ctypes.byref(a[0]), *a[1:]))  # noqa: E731
    # L <= 64 tile kernels read fp32 bias/mask directly: no table, no forward workspace
    d49 = _desc_v2(64, 3, 49, 32, mask_windows=4)
    assert q("fwa_add_table_bytes", d49, 1, 1) == 0
    assert q("fwa_fwd_workspace_bytes", d49, 1, 1) == 0
    # L = 144 flat kernels: f16 (bias + mask) * log2e table [n_w][h][L][L], 256-byte rounded
    d144 = _desc_v2(256, 16, 144, 32, mask_windows=4)
    tab = ((4 * 16 * 144 * 144 * 2 + 255) // 256) * 256
    assert q("fwa_add_table_bytes", d144, 1, 1) == tab
    assert q("fwa_fwd_workspace_bytes", d144, 1, 1) == tab
    assert q("fwa_fwd_workspace_bytes", d144, 1, 0) == ((16 * 144 * 144 * 2 + 255) // 256) * 256
    assert q("fwa_fwd_workspace_bytes", d144, 0, 0) == 0
    # backward: table + per-CTA dBias partials (f16 here: fp32 slices would exceed L2 / 2)
    ws = q("fwa_bwd_workspace_bytes", d144, 1, 1, 1)
    assert ws > tab and (ws - tab) % (144 * 144 * 2) == 0
    assert q("fwa_bwd_workspace_bytes", d144, 1, 1, 0) == tab
    # a prebuilt table (desc.add_table) removes it from both queries
    d144.add_table = 1 << 20
    assert q("fwa_fwd_workspace_bytes", d144, 1, 1) == 0
    assert q("fwa_bwd_workspace_bytes", d144, 1, 1, 1) == ws - tab


def test_shard_fill_offsets_follow_the_counter_based_stream():
    # fill_uniform_at(state, offset) must equal the slice of one fill_uniform draw: the
    # per-rank shard of bench.py's validation (checked on the oracle's generator, no GPU)
    from oracle import flashwin_oracle as orc

    whole = orc.fill_uniform(orc.Rng(42), (10, 6))
    state = 42 + 7 * 0x9E3779B97F4A7C15
    part = orc.splitmix_u64(state & ((1 << 64) - 1), 12)
    assert np.array_equal((part >> 11) * 2.0 ** -53 * 2.0 - 1.0, whole.reshape(-1)[7:19])


def test_abi2_error_paths_fail_before_any_device_work():
    # CAPACITY / SHAPE are raised by validation, before anything is enqueued (fake pointers
    # are never dereferenced): the reference's "check before work" order (flash.py:156)
    lib = nat.load()
    before = lib.fwa_launch_count()
    d = _desc_v2(64, 4, 144, 32)
    fake = ctypes.c_void_p(0x1000)
    # bias/mask on the large-window kernels without workspace for the add table
    assert lib.fwa_fwd(ctypes.byref(d), fake, fake, fake, fake, None, fake, None, 0, None) == 2
    assert b"workspace" in lib.fwa_last_error()
    # a table needs a bias or a mask, and enough bytes
    assert lib.fwa_build_add_table(ctypes.byref(d), None, None, fake, 1 << 30, None) == 1
    assert lib.fwa_build_add_table(ctypes.byref(d), fake, None, fake, 16, None) == 2
    # backward with dBias and a too-small workspace
    n = int(lib.fwa_bwd_workspace_bytes(ctypes.byref(d), 1, 0, 1))
    assert n > 0
    st = lib.fwa_bwd(ctypes.byref(d), fake, fake, fake, fake, fake, None, fake, fake, fake, fake,
                     fake, ctypes.c_size_t(n - 256), None)
    assert st == 2
    assert lib.fwa_launch_count() == before
