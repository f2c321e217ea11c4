"""The reference's own test_flash.py / test_acceptance.py cases, run against the drop-in API.

Same calls, same assertions (traffic, peaks, context identity, errors), with
the numeric tolerance moved from the reference's float64 1e-10 to the north
star's fp32 1e-5 relative (the GPU computes float64 host inputs in fp32).
"""

import numpy as np
import pytest
import torch

from oracle import flashwin_oracle as orc

pytestmark = pytest.mark.gpu

fw = pytest.importorskip("paper_2501_06480_b200")
from paper_2501_06480_b200 import (  # noqa: E402
    CapacityError,
    ContextError,
    FlashContext,
    InvalidRangeError,
    ScratchpadArena,
    ShapeError,
    TileConfig,
    batched_flash_backward,
    batched_flash_forward,
    flash_backward,
    flash_forward,
    peak_sram_backward,
    peak_sram_forward,
)

TOL = 1e-5


def rel_err(a, b):
    a = np.asarray(a.array if hasattr(a, "array") else a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def make_qkv(seed, L, C, n=3):
    rng = orc.Rng(seed)
    return tuple(orc.fill_uniform(rng, (L, C)) for _ in range(n))


@pytest.mark.parametrize("L,C", [(1, 16), (2, 16), (8, 32), (49, 32), (64, 64)])
@pytest.mark.parametrize("r", [1, 2, 4])
def test_forward_matches_oracle_with_exact_traffic_and_peak(L, C, r):
    q, k, v = make_qkv(40 + L + C + r, L, C)
    cfg = TileConfig(r=r)
    arena = ScratchpadArena()
    o, ctx, report = flash_forward(q, k, v, cfg, arena)
    o_ref, _ = orc.attention_forward(q, k, v)
    assert rel_err(o, o_ref) <= TOL
    assert isinstance(o, np.ndarray) and o.dtype == np.float64
    assert report.loads == {"Q": L * C, "K": L * C, "V": L * C}
    assert report.stores == {"O": L * C}
    assert report.peak_sram_bytes == peak_sram_forward(L, C, cfg)
    assert arena.live_bytes == 0
    assert ctx.q is q and ctx.k is k and ctx.v is v


@pytest.mark.parametrize("L,C", [(1, 16), (2, 16), (8, 32), (49, 32), (64, 64)])
@pytest.mark.parametrize("r", [1, 2, 4])
def test_backward_matches_analytic_oracle(L, C, r):
    rng = orc.Rng(50 + L + C + r)
    q, k, v, do = (orc.fill_uniform(rng, (L, C)) for _ in range(4))
    cfg = TileConfig(r=r)
    _, ctx, _ = flash_forward(q, k, v, cfg, ScratchpadArena())
    arena = ScratchpadArena()
    dq, dk, dv, report = flash_backward(ctx, do, arena)
    _, p = orc.attention_forward(q, k, v)
    ndq, ndk, ndv = orc.attention_backward(q, k, v, p, do)
    assert rel_err(dq, ndq) <= TOL and rel_err(dk, ndk) <= TOL and rel_err(dv, ndv) <= TOL
    assert report.loads == {"Q": 2 * L * C, "K": 2 * L * C, "V": L * C, "dO": L * C}
    assert report.stores == {"dQ": L * C, "dK": L * C, "dV": L * C}
    assert report.kernel_loads == {"Q": L * C, "K": L * C, "V": L * C, "dO": L * C}
    assert report.peak_sram_bytes == peak_sram_backward(L, C, cfg)
    assert arena.live_bytes == 0


def test_zero_keys_give_column_means_for_any_r():
    rng = orc.Rng(43)
    q, v = orc.fill_uniform(rng, (6, 8)), orc.fill_uniform(rng, (6, 8))
    means = np.tile(v.mean(axis=0), (6, 1))
    for r in (1, 2, 4):
        o, _, _ = flash_forward(q, np.zeros((6, 8)), v, TileConfig(r=r), ScratchpadArena())
        assert np.abs(o - means).max() <= 1e-6


def test_ragged_chunks_still_match_oracle():
    q, k, v = make_qkv(44, 8, 10)
    cfg = TileConfig(r=4)
    o, _, report = flash_forward(q, k, v, cfg, ScratchpadArena())
    assert rel_err(o, orc.attention_forward(q, k, v)[0]) <= TOL
    assert report.loads == {"Q": 80, "K": 80, "V": 80}
    assert report.peak_sram_bytes == peak_sram_forward(8, 10, cfg)


def test_scale_propagates_like_the_oracle():
    q, k, v = make_qkv(45, 8, 16)
    o, _, _ = flash_forward(q, k, v, TileConfig(r=2, scale=0.25), ScratchpadArena())
    assert rel_err(o, orc.attention_forward(q, k, v, 0.25)[0]) <= TOL


def test_large_window_exceeds_default_budget():
    q, k, v = make_qkv(46, 1024, 32)
    with pytest.raises(CapacityError) as exc:
        flash_forward(q, k, v, TileConfig(r=2, elem_bytes=4), ScratchpadArena(131072))
    msg = str(exc.value)
    assert "131072" in msg
    assert str(peak_sram_forward(1024, 32, TileConfig(r=2, elem_bytes=4))) in msg
    # with a large enough budget the GPU path runs L=1024 (generic kernel)
    o, _, _ = flash_forward(q, k, v, TileConfig(r=2), ScratchpadArena(1 << 24))
    assert rel_err(o, orc.attention_forward(q, k, v)[0]) <= TOL


def test_shape_and_context_errors():
    with pytest.raises(ShapeError):
        flash_forward(np.zeros((2, 4)), np.zeros((2, 4)), np.zeros((2, 6)), TileConfig(r=1),
                      ScratchpadArena())
    q, k, v = make_qkv(55, 4, 8)
    _, ctx, _ = flash_forward(q, k, v, TileConfig(r=2), ScratchpadArena())
    with pytest.raises(ShapeError):
        flash_backward(ctx, np.zeros((4, 6)), ScratchpadArena())
    with pytest.raises(ContextError):
        flash_backward(None, np.zeros((2, 2)), ScratchpadArena())
    with pytest.raises(ContextError):
        flash_backward(FlashContext(q=None, k=None, v=None, cfg=TileConfig(r=1)),
                       np.zeros((2, 2)), ScratchpadArena())


def test_budget_enforced_before_any_work():
    q, k, v = make_qkv(56, 16, 16)
    cfg = TileConfig(r=1, elem_bytes=8)
    _, ctx, _ = flash_forward(q, k, v, cfg, ScratchpadArena())
    small = ScratchpadArena(peak_sram_backward(16, 16, cfg) - 1)
    before = fw._native.launch_count()
    with pytest.raises(CapacityError):
        flash_backward(ctx, np.zeros((16, 16)), small)
    assert small.live_bytes == 0
    assert fw._native.launch_count() == before  # no kernel was enqueued


@pytest.mark.parametrize("L,C", [(8, 16), (49, 32), (64, 64)])
def test_outputs_and_gradients_agree_across_r(L, C):
    rng = orc.Rng(60)
    q, k, v, do = (orc.fill_uniform(rng, (L, C)) for _ in range(4))
    outs, grads = [], []
    for r in (1, 2, 4, 8):
        o, ctx, _ = flash_forward(q, k, v, TileConfig(r=r), ScratchpadArena())
        outs.append(o)
        grads.append(flash_backward(ctx, do, ScratchpadArena())[:3])
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)  # r is a tiling hint: bitwise invariant on B200
    for g in grads[1:]:
        for a, b in zip(grads[0], g):
            assert np.array_equal(a, b)


class TestBatched:
    def test_merged_counts_scale_with_slices(self):
        rng = orc.Rng(70)
        q, k, v = (orc.fill_uniform(rng, (4, 4, 64, 64)) for _ in range(3))
        _, _, report = batched_flash_forward(q, k, v, TileConfig(r=4), [ScratchpadArena()])
        assert report.loads["Q"] == 65536 and report.stores["O"] == 65536
        assert report.peak_sram_bytes == 24576

    def test_every_slice_matches_the_oracle(self):
        rng = orc.Rng(72)
        q, k, v = (orc.fill_uniform(rng, (2, 4, 64, 16)) for _ in range(3))
        out, ctxs, _ = batched_flash_forward(q, k, v, TileConfig(r=1), [ScratchpadArena()])
        assert rel_err(out, orc.attention_forward(q, k, v)[0]) <= TOL
        assert len(ctxs) == 2 and len(ctxs[0]) == 4
        assert np.array_equal(ctxs[1][2].q, q[1, 2])

    def test_worker_count_does_not_change_results(self):
        rng = orc.Rng(73)
        q, k, v = (orc.fill_uniform(rng, (3, 2, 16, 16)) for _ in range(3))
        cfg = TileConfig(r=2)
        out1, _, rep1 = batched_flash_forward(q, k, v, cfg, [ScratchpadArena()])
        out3, _, rep3 = batched_flash_forward(q, k, v, cfg, [ScratchpadArena() for _ in range(3)])
        assert np.array_equal(out1, out3)
        assert rep1.loads == rep3.loads and rep1.peak_sram_bytes == rep3.peak_sram_bytes

    def test_failures_name_the_slice(self):
        rng = orc.Rng(74)
        q, k, v = (orc.fill_uniform(rng, (2, 2, 64, 64)) for _ in range(3))
        with pytest.raises(CapacityError, match=r"slice \(b=0, head=0\)"):
            batched_flash_forward(q, k, v, TileConfig(r=1), [ScratchpadArena(1024)])

    def test_requires_4d_inputs_and_an_arena(self):
        rng = orc.Rng(75)
        q, k, v = (orc.fill_uniform(rng, (4, 8)) for _ in range(3))
        with pytest.raises(ShapeError):
            batched_flash_forward(q, k, v, TileConfig(r=1), [ScratchpadArena()])
        q4, k4, v4 = (orc.fill_uniform(rng, (1, 1, 4, 8)) for _ in range(3))
        with pytest.raises(InvalidRangeError):
            batched_flash_forward(q4, k4, v4, TileConfig(r=1), [])

    def test_batched_backward_on_device_tensors(self):
        shape = (16, 3, 49, 32)
        rng = fw.Rng(3)
        q, k, v, do = (fw.fill_uniform(rng, shape, dtype=torch.float16) for _ in range(4))
        cfg = TileConfig(r=2, scale=32 ** -0.5)
        o, ctxs, _ = batched_flash_forward(q, k, v, cfg, [ScratchpadArena()])
        assert o.is_cuda and o.dtype == torch.float16
        dq, dk, dv, rep = batched_flash_backward(ctxs, do, [ScratchpadArena()])
        qh, kh, vh, doh = (t.double().cpu().numpy() for t in (q, k, v, do))
        _, p = orc.attention_forward(qh, kh, vh, cfg.scale)
        for got, ref in zip((dq, dk, dv), orc.attention_backward(qh, kh, vh, p, doh, cfg.scale)):
            assert np.abs(got.double().cpu().numpy() - ref).max() <= 2e-2
        assert rep.loads["dO"] == 16 * 3 * 49 * 32


def test_torch_cpu_and_cuda_inputs_round_trip():
    rng = orc.Rng(9)
    q, k, v = (torch.from_numpy(orc.fill_uniform(rng, (8, 16))).float() for _ in range(3))
    o, _, _ = flash_forward(q, k, v, TileConfig(r=1), ScratchpadArena())
    assert o.device.type == "cpu" and o.dtype == torch.float32
    o2, _, _ = flash_forward(q.cuda(), k.cuda(), v.cuda(), TileConfig(r=1), ScratchpadArena())
    assert o2.is_cuda and torch.equal(o2.cpu(), o)


class _Dense:
    """DenseTensor surface (tensor.py:26-71): read-only ``.array``, no ``__getitem__``."""

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


def test_harness_fwd_bwd_pattern_on_dense_tensors():
    # replays harness.py:_time_flash (fwd_bwd): batched forward, then flash_backward on
    # contexts[b][head] with a DenseTensor dO slice per (b, head)
    B, h, L, C = 2, 3, 49, 32
    rng = orc.Rng(42)
    q, k, v, do = (_Dense((B, h, L, C), orc.fill_uniform(rng, (B, h, L, C))) for _ in range(4))
    cfg = TileConfig(r=2, scale=C ** -0.5)
    arena = ScratchpadArena()
    out, contexts, _ = batched_flash_forward(q, k, v, cfg, [arena])
    ref_o, p = orc.attention_forward(q.array, k.array, v.array, cfg.scale)
    assert rel_err(out.array, ref_o) <= TOL
    rq, rk, rv = orc.attention_backward(q.array, k.array, v.array, p, do.array, cfg.scale)
    for b in range(B):
        for head in range(h):
            sl_do = _Dense((L, C), do.array[b, head])
            dq, dk, dv, _ = flash_backward(contexts[b][head], sl_do, arena)
            for got, want in zip((dq, dk, dv), (rq[b, head], rk[b, head], rv[b, head])):
                assert rel_err(got.array, want) <= TOL


def test_slice_backward_keeps_the_forward_bias_and_mask():
    # a slice's context must differentiate the biased / masked attention the batched
    # forward ran, not plain attention
    B, h, L, C, nW = 4, 2, 49, 32, 2
    rng = fw.Rng(11)
    q, k, v, do = (fw.fill_uniform(rng, (B, h, L, C), dtype=torch.float16) for _ in range(4))
    bias = fw.fill_uniform(rng, (h, L, L), -2.0, 2.0)
    mask = torch.where(fw.fill_uniform(rng, (nW, L, L)) > 0.5, -100.0, 0.0).float().contiguous()
    cfg = TileConfig(r=2, scale=C ** -0.5)
    _, ctxs, _ = batched_flash_forward(q, k, v, cfg, [ScratchpadArena()], bias=bias, mask=mask)
    dq, dk, dv, _ = batched_flash_backward(ctxs, do, [ScratchpadArena()])
    for b in range(B):
        for head in range(h):
            c = ctxs[b][head]
            sq, sk, sv, _ = flash_backward(c, do[b, head], ScratchpadArena())
            for got, want in zip((sq, sk, sv), (dq[b, head], dk[b, head], dv[b, head])):
                assert (got.float() - want.float()).abs().max().item() <= 2e-2
