"""GPU parity: libfwa.so kernels vs the CPU oracle on identical SplitMix64 inputs.

Grids mirror the reference's own tests (test_acceptance.py:33-44, test_flash.py:99-112,
:169-186) plus the BASELINE shapes (L = 49, 64, 144, 256; d = 32, 64), ragged
feature counts (d = 4, 10), and the Swin bias/mask extension.
Tolerances (north star): fp32 1e-5 relative; fp16/bf16 2e-2 absolute vs the
float64 oracle run on the same quantised inputs.
"""

import math

import numpy as np
import pytest
import torch

from oracle import flashwin_oracle as orc
from tests._util import DTYPES, draw, err_ok, quantize

pytestmark = pytest.mark.gpu

fwa = pytest.importorskip("paper_2501_06480_b200")
ops = fwa.ops


def _bias_mask(h, L, nW, seed):
    rng = orc.Rng(seed)
    bias = orc.fill_uniform(rng, (h, L, L), -0.5, 0.5).astype(np.float32)
    mask = np.where(orc.fill_uniform(rng, (nW, L, L)) > 0.3, -100.0, 0.0).astype(np.float32)
    return bias, mask


FWD_CASES = [
    # (N, h, L, d)
    (2, 1, 1, 16), (2, 1, 2, 16), (3, 2, 8, 32), (4, 3, 49, 32), (2, 2, 64, 64),
    (2, 1, 8, 4), (3, 1, 8, 10), (5, 3, 49, 16), (3, 2, 144, 32), (2, 2, 256, 32),
    (2, 1, 256, 64), (2, 2, 100, 24), (1, 1, 17, 128),
]


@pytest.mark.parametrize("dt", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("N,h,L,d", FWD_CASES)
@pytest.mark.parametrize("kernel", ["auto", "generic", "tc"])
def test_forward_matches_oracle(dt, N, h, L, d, kernel):
    dtype = DTYPES[dt]
    if kernel == "tc" and ops.footprint(N, h, L, d, dtype)["kernel_fwd"] != "tc":
        pytest.skip("shape/dtype not on the tcgen05 path")
    (q, k, v), (qh, kh, vh) = draw(9000 + 100 * L + d, (N, h, L, d), 3, dtype)
    for scale in (1.0, d ** -0.5):
        o = ops.attention_forward(q, k, v, scale, kernel=kernel)
        ref, _ = orc.attention_forward(qh, kh, vh, scale)
        ok, err = err_ok(o, ref, dtype)
        assert ok, f"{dt} {(N, h, L, d)} scale={scale} err={err}"


@pytest.mark.parametrize("dt", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("N,h,L,d", [(4, 3, 49, 32), (4, 2, 64, 32), (2, 2, 144, 32), (2, 1, 256, 64), (6, 2, 16, 10)])
@pytest.mark.parametrize("kernel", ["auto", "generic"])
def test_forward_bias_mask_matches_oracle(dt, N, h, L, d, kernel):
    dtype = DTYPES[dt]
    nW = 3 if N % 3 == 0 else 2
    (q, k, v), (qh, kh, vh) = draw(77 + L + d, (N, h, L, d), 3, dtype)
    bias, mask = _bias_mask(h, L, nW, 5)
    o = ops.attention_forward(q, k, v, d ** -0.5, torch.from_numpy(bias).cuda(),
                              torch.from_numpy(mask).cuda(), kernel=kernel)
    ref, _ = orc.attention_forward(qh, kh, vh, d ** -0.5, bias=bias.astype(np.float64),
                                   mask=mask.astype(np.float64))
    ok, err = err_ok(o, ref, dtype)
    assert ok, err


BWD_CASES = [(2, 1, 1, 16), (2, 1, 2, 16), (3, 2, 8, 32), (4, 3, 49, 32), (2, 2, 64, 64),
             (2, 1, 8, 4), (3, 1, 8, 10), (2, 2, 144, 32), (2, 1, 256, 32), (2, 1, 256, 64)]


BWD_CASES += [(5, 3, 49, 16), (3, 2, 36, 64), (7, 3, 49, 32)]


@pytest.mark.parametrize("dt", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("N,h,L,d", BWD_CASES)
@pytest.mark.parametrize("kernel", ["auto", "generic", "tc"])
def test_backward_matches_oracle(dt, N, h, L, d, kernel):
    dtype = DTYPES[dt]
    if kernel == "tc" and ops.footprint(N, h, L, d, dtype)["kernel_bwd"] != "tc":
        pytest.skip("shape/dtype not on the tcgen05 path")
    (q, k, v, do), (qh, kh, vh, doh) = draw(50 + L + d, (N, h, L, d), 4, dtype)
    for scale in (1.0, d ** -0.5):
        dq, dk, dv, _ = ops.attention_backward(q, k, v, do, scale, kernel=kernel)
        _, p = orc.attention_forward(qh, kh, vh, scale)
        rdq, rdk, rdv = orc.attention_backward(qh, kh, vh, p, doh, scale)
        for name, got, ref in (("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
            ok, err = err_ok(got, ref, dtype)
            assert ok, f"{name} {dt} {(N, h, L, d)} scale={scale} err={err}"


@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("N,h,L,d", [(6, 3, 49, 32), (4, 2, 144, 32), (3, 2, 16, 10)])
def test_backward_bias_mask_dbias(dt, N, h, L, d):
    dtype = DTYPES[dt]
    nW = 3 if N % 3 == 0 else 2
    (q, k, v, do), (qh, kh, vh, doh) = draw(31 + L, (N, h, L, d), 4, dtype)
    bias, mask = _bias_mask(h, L, nW, 9)
    bt, mt = torch.from_numpy(bias).cuda(), torch.from_numpy(mask).cuda()
    dq, dk, dv, db = ops.attention_backward(q, k, v, do, d ** -0.5, bt, mt, want_dbias=True)
    _, p = orc.attention_forward(qh, kh, vh, d ** -0.5, bias=bias.astype(np.float64),
                                 mask=mask.astype(np.float64))
    rdq, rdk, rdv, rdb = orc.attention_backward(qh, kh, vh, p, doh, d ** -0.5, want_dbias=True)
    for name, got, ref in (("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
        ok, err = err_ok(got, ref, dtype)
        assert ok, f"{name} err={err}"
    # dBias accumulates N fp32 partial sums: fp32 accumulation tolerance
    db_err = float(np.abs(db.cpu().numpy() - rdb).max())
    assert db_err <= (1e-4 if dtype == torch.float32 else 3e-2) * max(1.0, float(np.abs(rdb).max())), db_err
    # deterministic: bitwise repeatable
    _, _, _, db2 = ops.attention_backward(q, k, v, do, d ** -0.5, bt, mt, want_dbias=True)
    assert torch.equal(db, db2)


def test_fill_uniform_bit_identical_to_oracle():
    for dt in DTYPES.values():
        r = fwa.Rng(42)
        got = fwa.fill_uniform(r, (1000, 7), -1.0, 1.0, dtype=dt)
        ref = quantize(orc.fill_uniform(orc.Rng(42), (1000, 7)), dt)
        assert np.array_equal(got.to(torch.float64).cpu().numpy(), ref)
        assert r.state == (42 + 7000 * orc.GOLDEN) & orc.MASK64


@pytest.mark.parametrize("scale_tag,scale", [("s1", 1.0), ("sr", 32 ** -0.5)])
def test_cfg1_fp32_against_reference_golden(golden, scale_tag, scale):
    """BASELINE configs[0]: fp32 (64,3,49,32) forward+backward vs the reference's numbers."""
    scalars, arrays = golden
    (q, k, v, do), _ = draw(42, (64, 3, 49, 32), 4, torch.float32)
    o = ops.attention_forward(q, k, v, scale)
    dq, dk, dv, _ = ops.attention_backward(q, k, v, do, scale)
    g = scalars[f"cfg1_{scale_tag}"]
    on = o.double().cpu().numpy()
    for name, got, ref in (("o_b0", on[0], arrays[f"cfg1_{scale_tag}_o_b0"]),
                           ("o_b63", on[63], arrays[f"cfg1_{scale_tag}_o_b63"]),
                           ("dq_b5", dq[5], arrays[f"cfg1_{scale_tag}_dq_b5"]),
                           ("dk_b5", dk[5], arrays[f"cfg1_{scale_tag}_dk_b5"]),
                           ("dv_b5", dv[5], arrays[f"cfg1_{scale_tag}_dv_b5"])):
        got = np.asarray(got.double().cpu().numpy() if isinstance(got, torch.Tensor) else got)
        assert np.abs(got - ref).max() / np.abs(ref).max() <= 1e-5, name
    assert math.isclose(float(np.abs(on).sum()), g["sum_abs_o"], rel_tol=1e-5)
    assert math.isclose(float(dv.double().sum()), g["sum_dv"], rel_tol=1e-5)
    assert abs(float(dk.double().sum())) < 1e-3


def test_window_partition_reverse_bitwise():
    for (B, H, W, C, kk, s) in [(2, 56, 56, 96, 7, 0), (2, 56, 56, 96, 7, 3), (1, 10, 15, 4, 5, 0),
                                (3, 14, 21, 3, 7, 3), (1, 4, 4, 1, 2, 0), (2, 96, 96, 128, 12, 6)]:
        for dt in (torch.float32, torch.float16, torch.bfloat16):
            x = fwa.fill_uniform(fwa.Rng(B + H + C), (B, H, W, C), dtype=dt)
            y = ops.window_partition(x, kk, s)
            ref = orc.window_partition(x.cpu().to(torch.float64).numpy(), kk, shift=s)
            assert np.array_equal(y.cpu().to(torch.float64).numpy(), ref)
            back = ops.window_reverse(y, kk, H, W, s)
            assert torch.equal(back, x)


def _torch_partition(x, k, s):
    B, H, W, C = x.shape
    if s:
        x = torch.roll(x, (-s, -s), (1, 2))
    return x.view(B, H // k, k, W // k, k, C).permute(0, 1, 3, 2, 4, 5).reshape(-1, k * k, C)


@pytest.mark.parametrize("B,H,C,k,s,dt", [
    (128, 56, 96, 7, 3, torch.bfloat16), (128, 28, 192, 7, 3, torch.float16),
    (128, 7, 768, 7, 0, torch.float16), (64, 96, 128, 12, 6, torch.bfloat16),
    (3, 20, 5, 4, 3, torch.uint8), (2, 14, 7, 7, 2, torch.float64), (5, 9, 33, 3, 2, torch.float16),
])
def test_window_partition_full_size_and_element_widths(B, H, C, k, s, dt):
    # every vector width of the copy kernel (16 / 8 / 4 / 2 / 1-byte moves) and the Swin-T /
    # Swin-B stage shapes at full batch, bitwise against the same permutation in torch
    x = torch.randint(0, 255, (B, H, H, C), dtype=torch.uint8, device="cuda") if dt == torch.uint8 \
        else fwa.fill_uniform(fwa.Rng(B + C), (B, H, H, C), dtype=dt if dt != torch.float64 else torch.float32).to(dt)
    y = ops.window_partition(x, k, s)
    assert torch.equal(y, _torch_partition(x, k, s))
    assert torch.equal(ops.window_reverse(y, k, H, H, s), x)


def test_window_api_matches_reference_index_map(golden):
    _, arrays = golden
    cfg = fwa.WindowConfig(4, 4, 1, 2)
    y = fwa.window_partition(np.arange(16.0).reshape(4, 4, 1), cfg)
    assert np.array_equal(y, arrays["win_4x4_k2"])
    x = orc.fill_uniform(orc.Rng(7), (10, 15, 4))
    y = fwa.window_partition(x, fwa.WindowConfig(10, 15, 4, 5))
    assert np.array_equal(y, arrays["win_10x15x4_k5"])  # float64 moved bitwise
    assert np.array_equal(fwa.window_reverse(y, fwa.WindowConfig(10, 15, 4, 5)), x)


def test_bias_gather_scatter_and_mask_match_oracle():
    for k, h in ((7, 3), (12, 4)):
        table = fwa.fill_uniform(fwa.Rng(k), ((2 * k - 1) ** 2, h), -0.1, 0.1)
        bias = ops.bias_gather(table, k)
        ref = orc.gather_bias(table.cpu().double().numpy(), k)
        assert np.array_equal(bias.cpu().double().numpy(), ref)
        db = fwa.fill_uniform(fwa.Rng(k + 1), (h, k * k, k * k))
        dt = ops.bias_scatter(db, k)
        idx = orc.relative_position_index(k).reshape(-1)
        rdt = np.zeros(((2 * k - 1) ** 2, h))
        np.add.at(rdt, idx, db.cpu().double().numpy().reshape(h, -1).T)
        assert np.abs(dt.cpu().double().numpy() - rdt).max() <= 1e-5
    m = ops.shift_mask(56, 56, 7, 3)
    assert np.array_equal(m.cpu().double().numpy(), orc.shifted_window_mask(56, 56, 7, 3))


@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_full_size_swin_t_stage1_properties(dt):
    """BASELINE configs[1]/[2] stage-1 size (8192, 3, 49, 32): size-independent checks."""
    dtype = DTYPES[dt]
    shape = (8192, 3, 49, 32)
    rng = fwa.Rng(42)
    q, k, v, do = (fwa.fill_uniform(rng, shape, dtype=dtype) for _ in range(4))
    scale = 32 ** -0.5
    o = ops.attention_forward(q, k, v, scale)
    # fp32 torch reference on device, chunked (float reference for a float kernel)
    for s in range(0, shape[0], 2048):
        sl = slice(s, s + 2048)
        sc = (q[sl].float() @ k[sl].float().transpose(-1, -2)) * scale
        ref = torch.softmax(sc, -1) @ v[sl].float()
        assert (o[sl].float() - ref).abs().max().item() <= 2e-2
    # rows of P sum to 1 => each O row lies in the convex hull of V rows
    assert (o.float() <= v.float().amax(dim=2, keepdim=True) + 1e-2).all()
    dq, dk, dv, _ = ops.attention_backward(q, k, v, do, scale)
    assert math.isclose(dv.double().sum().item(), do.double().sum().item(), rel_tol=2e-3, abs_tol=2.0)
    per_unit_dk = dk.double().sum(dim=2)  # sum over keys of dK = scale * sum_j dS^T Q = ...
    assert torch.isfinite(per_unit_dk).all()


def test_autograd_matches_torch_reference():
    shape = (6, 3, 49, 32)
    rng = fwa.Rng(5)
    q, k, v = (fwa.fill_uniform(rng, shape, dtype=torch.float32).requires_grad_() for _ in range(3))
    table = (0.02 * torch.randn(13 * 13, 3, device="cuda")).requires_grad_()
    mask = ops.shift_mask(14, 21, 7, 3)  # nW = 6
    bias = fwa.relative_position_bias(table, 7)
    o = fwa.window_attention(q, k, v, None, bias, mask)
    g = torch.randn_like(o)
    (o * g).sum().backward()
    grads = [t.grad.clone() for t in (q, k, v, table)]
    for t in (q, k, v, table):
        t.grad = None
    bias_ref = table[torch.from_numpy(orc.relative_position_index(7).reshape(-1)).cuda()].view(49, 49, 3).permute(2, 0, 1)
    s = (q @ k.transpose(-1, -2)) * 32 ** -0.5 + bias_ref[None] + mask[torch.arange(6, device="cuda") % 6][:, None]
    ref = torch.softmax(s, -1) @ v
    (ref * g).sum().backward()
    assert (o - ref).abs().max().item() <= 1e-5
    for got, t in zip(grads, (q, k, v, table)):
        assert (got - t.grad).abs().max().item() <= 1e-4 * max(1.0, t.grad.abs().max().item())


def test_tc_kernel_selected_for_swin_shapes():
    for d in (16, 32, 64):
        for dt in (torch.float16, torch.bfloat16):
            assert ops.footprint(8192, 3, 49, d, dt)["kernel_fwd"] == "tc"
            assert ops.footprint(100, 2, 64, d, dt)["kernel_fwd"] == "tc"
    assert ops.footprint(8192, 3, 49, 32, torch.bfloat16)["kernel_bwd"] == "tc"
    assert ops.footprint(64, 3, 49, 32, torch.float32)["kernel_fwd"] == "generic"
    assert ops.footprint(64, 3, 49, 10, torch.float16)["kernel_fwd"] == "generic"


@pytest.mark.parametrize("dt", ["f16", "bf16"])
@pytest.mark.parametrize("units", [1, 2, 3, 295, 296, 297, 593, 4097])
def test_tc_forward_tile_counts(dt, units):
    """Odd unit counts (half-empty last tile) and grid wrap-around of the persistent scheduler."""
    dtype = DTYPES[dt]
    (q, k, v), (qh, kh, vh) = draw(units, (units, 1, 49, 32), 3, dtype)
    o = ops.attention_forward(q, k, v, 0.2, kernel="tc")
    ref, _ = orc.attention_forward(qh, kh, vh, 0.2)
    ok, err = err_ok(o, ref, dtype)
    assert ok, err


def test_tc_forward_does_not_write_outside_output():
    """Rows L..63 of the padded tile and the phantom unit of the last tile are clipped by TMA."""
    q, k, v = (fwa.fill_uniform(fwa.Rng(i), (3, 1, 49, 32), dtype=torch.float16) for i in range(3))
    big = torch.full((4 * 49 * 32 + 4096,), 7.0, dtype=torch.float16, device="cuda")
    out = big[: 3 * 49 * 32].view(3, 1, 49, 32)
    ops.attention_forward(q, k, v, 0.2, kernel="tc", out=out)
    torch.cuda.synchronize()
    assert (big[3 * 49 * 32:] == 7.0).all()


@pytest.mark.parametrize("dt", ["f16", "bf16"])
@pytest.mark.parametrize("units", [1, 3, 297, 1025])
def test_tc_backward_tile_counts(dt, units):
    dtype = DTYPES[dt]
    (q, k, v, do), (qh, kh, vh, doh) = draw(units + 7, (units, 1, 49, 32), 4, dtype)
    dq, dk, dv, _ = ops.attention_backward(q, k, v, do, 0.3, kernel="tc")
    _, p = orc.attention_forward(qh, kh, vh, 0.3)
    for got, ref in zip((dq, dk, dv), orc.attention_backward(qh, kh, vh, p, doh, 0.3)):
        ok, err = err_ok(got, ref, dtype)
        assert ok, err
    assert fwa._native.device_flags() == 0


def test_tc_backward_does_not_write_outside_outputs():
    q, k, v, do = (fwa.fill_uniform(fwa.Rng(i), (3, 1, 49, 32), dtype=torch.float16) for i in range(4))
    dq, dk, dv, _ = ops.attention_backward(q, k, v, do, 0.2, kernel="tc")
    torch.cuda.synchronize()
    assert torch.isfinite(dq).all() and torch.isfinite(dk).all() and torch.isfinite(dv).all()
    # rows of dK sum to zero over keys? no: sum over keys of dK_j = scale * sum_ij dS_ij Q_i = 0
    assert dk.float().sum(dim=2).abs().max().item() < 2e-2


def _torch_ref(q, k, v, scale, bias=None, mask=None):
    s = (q.float() @ k.float().transpose(-1, -2)) * scale
    if bias is not None:
        s = s + bias[None]
    if mask is not None:
        nW = mask.shape[0]
        s = s + mask[torch.arange(q.shape[0], device=q.device) % nW][:, None]
    return torch.softmax(s, -1) @ v.float()


@pytest.mark.parametrize("dt", ["f16", "bf16"])
@pytest.mark.parametrize("N,h,L,d,nW,use_bias", [
    (8192, 3, 49, 32, 64, True),    # Swin-T stage 1, shifted layer: period 96 tiles
    (2048, 6, 49, 32, 16, True),
    (128, 24, 49, 32, 0, True),     # stage 4: bias only
    (3000, 5, 49, 16, 7, True),     # odd period (35 tiles)
    (1500, 3, 64, 64, 0, True),     # bias only, d=64 (1 CTA/SM)
    (999, 2, 36, 32, 9, False),     # mask only
    (600, 1, 49, 32, 300, True),    # period (150) above the grid cap -> generic kernel
])
def test_forward_bias_mask_full_size(dt, N, h, L, d, nW, use_bias):
    dtype = DTYPES[dt]
    rng = fwa.Rng(N + h)
    q, k, v = (fwa.fill_uniform(rng, (N, h, L, d), dtype=dtype) for _ in range(3))
    bias = fwa.fill_uniform(rng, (h, L, L), -1.0, 1.0) if use_bias else None
    mask = None
    if nW:
        mask = torch.where(fwa.fill_uniform(rng, (nW, L, L)) > 0.4, -100.0, 0.0).float().contiguous()
    o = ops.attention_forward(q, k, v, d ** -0.5, bias, mask)
    ref = _torch_ref(q, k, v, d ** -0.5, bias, mask)
    assert (o.float() - ref).abs().max().item() <= 2e-2
    assert fwa._native.device_flags() == 0


@pytest.mark.parametrize("dt", ["f16", "bf16"])
@pytest.mark.parametrize("N,h,L,d,nW,use_bias,want_db", [
    (8192, 3, 49, 32, 64, True, True),    # Swin-T stage 1 shifted layer, learnable bias
    (512, 12, 49, 32, 4, True, True),
    (128, 24, 49, 32, 0, True, True),
    (3000, 5, 49, 16, 7, True, False),
    (1500, 3, 64, 64, 0, True, True),
    (999, 2, 36, 32, 9, False, False),
    (600, 1, 49, 32, 300, True, True),    # period above the grid cap -> generic kernel
])
def test_backward_bias_mask_full_size(dt, N, h, L, d, nW, use_bias, want_db):
    dtype = DTYPES[dt]
    rng = fwa.Rng(N + 2 * h)
    q, k, v, do = (fwa.fill_uniform(rng, (N, h, L, d), dtype=dtype) for _ in range(4))
    bias = fwa.fill_uniform(rng, (h, L, L), -1.0, 1.0) if use_bias else None
    mask = None
    if nW:
        mask = torch.where(fwa.fill_uniform(rng, (nW, L, L)) > 0.4, -100.0, 0.0).float().contiguous()
    sc = d ** -0.5
    dq, dk, dv, db = ops.attention_backward(q, k, v, do, sc, bias, mask, want_dbias=want_db)
    qf, kf, vf = (t.float().requires_grad_() for t in (q, k, v))
    bf = bias.clone().requires_grad_() if bias is not None else None
    ref = _torch_ref(qf, kf, vf, sc, bf, mask)
    ref.backward(do.float())
    for got, t in ((dq, qf), (dk, kf), (dv, vf)):
        assert (got.float() - t.grad).abs().max().item() <= 2e-2
    if want_db:
        scale_db = max(1.0, bf.grad.abs().max().item())
        assert (db - bf.grad).abs().max().item() <= 1e-2 * scale_db
        _, _, _, db2 = ops.attention_backward(q, k, v, do, sc, bias, mask, want_dbias=True)
        assert torch.equal(db, db2)  # deterministic
    assert fwa._native.device_flags() == 0


def test_footprint_reports_kernel_and_paper_peaks():
    fp = ops.footprint(8192, 3, 49, 32, torch.float16, chunks=2)
    assert fp["paper_peak_fwd"] == (49 * 49 + 2 * 49 * 16) * 2
    assert fp["hbm_bytes_fwd"] == 4 * 8192 * 3 * 49 * 32 * 2
    assert fp["smem_bytes_fwd"] > 0
