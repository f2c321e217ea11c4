"""Flat-row large-window kernels (fwa_tc_flat.cu) on many units.

The flat forward packs 128-row blocks across unit boundaries and gives each CTA a
contiguous unit range, so the interesting cases are unit counts that leave ragged
ranges (not a multiple of the SM count), blocks holding 2-3 units (L < 128 or
L % 128 != 0) and the last, partial block of every range. Checked against a float32
torch restatement of the oracle's math (oracle/flashwin_oracle.py: softmax(QK^T s) V)
within the package's 16-bit tolerance.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu

fwa = pytest.importorskip("paper_2501_06480_b200")
ops = fwa.ops


def _ref(q, k, v, scale):
    s = (q.float() @ k.float().transpose(-1, -2)) * scale
    return torch.softmax(s, -1) @ v.float()


@pytest.mark.parametrize("dt", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("units,L,d", [
    (149, 144, 32), (301, 144, 32), (1000, 144, 32), (150, 80, 32), (151, 96, 16), (299, 112, 64),
    (148, 128, 32), (297, 160, 32), (160, 192, 16), (149, 208, 32), (300, 240, 32), (151, 256, 32),
    (149, 256, 64), (150, 144, 64), (7, 144, 32), (1, 256, 32),
])
def test_flat_forward_matches_fp32(dt, units, L, d):
    rng = fwa.Rng(units * 31 + L + d)
    shape = (units, 1, L, d)
    q, k, v = (fwa.fill_uniform(rng, shape, dtype=dt) for _ in range(3))
    scale = d ** -0.5
    o = ops.attention_forward(q, k, v, scale)
    ref = _ref(q, k, v, scale)
    err = (o.float() - ref).abs().max().item()
    assert err <= 2e-2, err
    assert torch.isfinite(o).all()
    assert fwa._native.device_flags() == 0


def test_flat_forward_heads_layout_is_flat_over_units():
    # (N, h) units are contiguous in [N][h][L][d]: heads change nothing for the flat kernel
    rng = fwa.Rng(5)
    q, k, v = (fwa.fill_uniform(rng, (37, 4, 144, 32), dtype=torch.float16) for _ in range(3))
    o = ops.attention_forward(q, k, v, 0.2)
    o_flat = ops.attention_forward(q.view(148, 1, 144, 32), k.view(148, 1, 144, 32),
                                   v.view(148, 1, 144, 32), 0.2)
    assert torch.equal(o.view(148, 1, 144, 32), o_flat)


def _ref_bwd(q, k, v, do, scale):
    qf, kf, vf = (t.float().requires_grad_(True) for t in (q, k, v))
    o = torch.softmax((qf @ kf.transpose(-1, -2)) * scale, -1) @ vf
    o.backward(do.float())
    return qf.grad, kf.grad, vf.grad


@pytest.mark.parametrize("dt", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("units,L,d", [
    (149, 144, 32), (301, 144, 32), (1000, 144, 32), (150, 80, 32), (151, 96, 16), (149, 112, 32),
    (148, 128, 32), (297, 160, 32), (160, 176, 32), (149, 208, 16), (150, 128, 64), (7, 144, 32),
    (1, 144, 32), (149, 256, 16), (149, 192, 32), (150, 240, 32), (151, 224, 16),
    # split K / V rings (kNeedKV K slots, one block's worth of V)
    (149, 256, 32), (1, 256, 32), (3, 256, 32), (151, 208, 32), (150, 96, 64), (149, 112, 64),
])
def test_flat_backward_matches_fp32(dt, units, L, d):
    rng = fwa.Rng(units * 17 + L + d)
    shape = (units, 1, L, d)
    q, k, v, do = (fwa.fill_uniform(rng, shape, dtype=dt) for _ in range(4))
    scale = d ** -0.5
    dq, dk, dv, _ = ops.attention_backward(q, k, v, do, scale)
    for got, want in zip((dq, dk, dv), _ref_bwd(q, k, v, do, scale)):
        err = (got.float() - want).abs().max().item()
        assert err <= 2e-2, err
        assert torch.isfinite(got).all()
    assert fwa._native.device_flags() == 0


def _ref_add(q, k, v, scale, bias, mask, heads):
    s = (q.float() @ k.float().transpose(-1, -2)) * scale
    N = q.shape[0]
    if bias is not None:
        s = s + bias[None]
    if mask is not None:
        s = s + mask[torch.arange(N, device=q.device) % mask.shape[0]][:, None]
    return torch.softmax(s, -1) @ v.float()


@pytest.mark.parametrize("dt", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("N,h,L,d,nw,with_bias", [
    (64, 4, 144, 32, 64, True), (37, 4, 144, 32, 4, True), (19, 8, 144, 32, 1, True),
    (64, 4, 144, 32, 16, False), (40, 2, 256, 32, 4, True), (33, 3, 80, 16, 3, True),
    (16, 4, 144, 64, 4, True),
])
def test_flat_forward_bias_mask_matches_fp32(dt, N, h, L, d, nw, with_bias):
    rng = fwa.Rng(N * 13 + L + nw)
    q, k, v = (fwa.fill_uniform(rng, (N, h, L, d), dtype=dt) for _ in range(3))
    bias = fwa.fill_uniform(rng, (h, L, L), -0.5, 0.5) if with_bias else None
    mask = torch.where(fwa.fill_uniform(rng, (nw, L, L)) > 0.6, -100.0, 0.0).float().contiguous() \
        if nw > 1 or not with_bias else None
    scale = d ** -0.5
    o = ops.attention_forward(q, k, v, scale, bias, mask)
    ref = _ref_add(q, k, v, scale, bias, mask, h)
    err = (o.float() - ref).abs().max().item()
    assert err <= 2e-2, err
    assert fwa._native.device_flags() == 0


def _ref_add_bwd(q, k, v, do, scale, bias, mask):
    qf, kf, vf = (t.float().requires_grad_(True) for t in (q, k, v))
    bf = bias.float().clone().requires_grad_(True) if bias is not None else None
    s = (qf @ kf.transpose(-1, -2)) * scale
    N = q.shape[0]
    if bf is not None:
        s = s + bf[None]
    if mask is not None:
        s = s + mask[torch.arange(N, device=q.device) % mask.shape[0]][:, None]
    (torch.softmax(s, -1) @ vf).backward(do.float())
    return qf.grad, kf.grad, vf.grad, (bf.grad if bf is not None else None)


@pytest.mark.parametrize("dt", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("N,h,L,nw,with_bias,want_db", [
    (64, 4, 144, 64, True, True), (37, 4, 144, 4, True, True), (19, 8, 144, 1, True, True),
    (64, 4, 144, 16, False, False), (33, 4, 144, 4, True, False), (24, 2, 96, 4, True, True),
    (10, 3, 256, 4, True, True), (9, 1, 144, 3, True, True),
])
def test_flat_backward_bias_mask_dbias_matches_fp32(dt, N, h, L, nw, with_bias, want_db):
    d = 32
    rng = fwa.Rng(N * 29 + L + nw)
    q, k, v, do = (fwa.fill_uniform(rng, (N, h, L, d), dtype=dt) for _ in range(4))
    bias = fwa.fill_uniform(rng, (h, L, L), -0.5, 0.5) if with_bias else None
    mask = torch.where(fwa.fill_uniform(rng, (nw, L, L)) > 0.6, -100.0, 0.0).float().contiguous() \
        if nw > 1 or not with_bias else None
    scale = d ** -0.5
    fp = ops.footprint(N, h, L, d, dt)
    assert fp["kernel_bwd"] == "tc"
    dq, dk, dv, db = ops.attention_backward(q, k, v, do, scale, bias, mask, want_dbias=want_db)
    rq, rk, rv, rb = _ref_add_bwd(q, k, v, do, scale, bias, mask)
    for got, want in zip((dq, dk, dv), (rq, rk, rv)):
        assert (got.float() - want).abs().max().item() <= 2e-2
    if want_db:
        tol = 2e-2 * max(1.0, rb.abs().max().item())
        assert (db - rb).abs().max().item() <= tol
    assert fwa._native.device_flags() == 0


def test_flat_backward_dbias_is_deterministic():
    rng = fwa.Rng(3)
    q, k, v, do = (fwa.fill_uniform(rng, (40, 4, 144, 32), dtype=torch.float16) for _ in range(4))
    bias = fwa.fill_uniform(rng, (4, 144, 144), -0.5, 0.5)
    outs = [ops.attention_backward(q, k, v, do, 0.2, bias, None, want_dbias=True)[3] for _ in range(6)]
    assert all(torch.equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("N,h", [(1024, 4), (256, 16)])
def test_flat_backward_dbias_first_touch_partials_are_deterministic(N, h):
    # >= heads units per CTA: each CTA's first unit of a head stores its partial rows, later
    # units reduce into them (no up-front zeroing); fp32 and f16 partials
    rng = fwa.Rng(N + h)
    q, k, v, do = (fwa.fill_uniform(rng, (N, h, 144, 32), dtype=torch.bfloat16) for _ in range(4))
    bias = fwa.fill_uniform(rng, (h, 144, 144), -1.0, 1.0)
    outs = [ops.attention_backward(q, k, v, do, 0.2, bias, None, want_dbias=True)[3] for _ in range(4)]
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    qf, kf, vf = (t.float().requires_grad_(True) for t in (q, k, v))
    bf = bias.clone().requires_grad_(True)
    (torch.softmax((qf @ kf.transpose(-1, -2)) * 0.2 + bf[None], -1) @ vf).backward(do.float())
    assert (outs[0] - bf.grad).abs().max().item() <= 2e-2 * max(1.0, bf.grad.abs().max().item())
