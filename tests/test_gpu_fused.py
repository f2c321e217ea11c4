"""Fused Swin layouts on the GPU.

* attention straight from the packed qkv-Linear output (N, L, 3*h*d) to the
  proj-Linear input (N, L, h*d): bitwise equal to split -> attention -> merge,
  because the same tcgen05 kernel does the math; only the TMA maps differ.
* a whole Swin (S)W-MSA block built from the package's kernels (cyclic shift +
  partition, qkv Linear, fused attention with relative-position bias and
  shift mask, proj Linear, reverse + unshift) against a plain fp32 torch
  implementation, forward and backward (x, weights, bias table).
"""

import math

import pytest
import torch

from oracle import flashwin_oracle as orc

pytestmark = pytest.mark.gpu

fwa = pytest.importorskip("paper_2501_06480_b200")
ops = fwa.ops


def _split_merge_reference(qkv, h, scale, bias, mask):
    N, L, C3 = qkv.shape
    d = C3 // (3 * h)
    q, k, v = (qkv.view(N, L, 3, h, d)[:, :, i].permute(0, 2, 1, 3).contiguous() for i in range(3))
    o = ops.attention_forward(q, k, v, scale, bias, mask)
    return o.permute(0, 2, 1, 3).reshape(N, L, h * d), (q, k, v)


@pytest.mark.parametrize("dt", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("N,h,L,d,extras", [
    (64, 3, 49, 32, False), (64, 3, 49, 32, True), (96, 6, 49, 32, True), (33, 4, 64, 16, False),
    (15, 5, 36, 64, True), (1, 3, 49, 32, False), (2048, 3, 49, 32, True),
    # Swin-B window 12 and the other pieces-mode windows (flat-row kernels, token-major maps)
    (64, 4, 144, 32, False), (64, 4, 144, 32, True), (256, 16, 144, 32, True), (7, 3, 144, 32, True),
    (20, 2, 256, 32, True), (9, 4, 128, 32, False), (12, 2, 192, 32, True),
])
def test_qkv_layout_bitwise_equal_to_split_path(dt, N, h, L, d, extras):
    rng = fwa.Rng(N * 7 + h)
    qkv = fwa.fill_uniform(rng, (N, L, 3 * h * d), dtype=dt)
    do = fwa.fill_uniform(rng, (N, L, h * d), dtype=dt)
    bias = mask = None
    if extras:
        k = int(math.isqrt(L))
        bias = fwa.fill_uniform(rng, (h, L, L), -0.3, 0.3)
        nW = 4 if N % 4 == 0 else 1
        mask = torch.where(fwa.fill_uniform(rng, (nW, L, L)) > 0.5, -100.0, 0.0).float().contiguous()
        del k
    sc = d ** -0.5
    o = ops.attention_forward_qkv(qkv, h, sc, bias, mask)
    ref, (q, k_, v) = _split_merge_reference(qkv, h, sc, bias, mask)
    assert torch.equal(o, ref)
    dqkv, db = ops.attention_backward_qkv(qkv, do, h, sc, bias, mask, want_dbias=bias is not None)
    do4 = do.view(N, L, h, d).permute(0, 2, 1, 3).contiguous()
    dq, dk, dv, db_ref = ops.attention_backward(q, k_, v, do4, sc, bias, mask, want_dbias=bias is not None)
    ref_dqkv = torch.stack([t.permute(0, 2, 1, 3) for t in (dq, dk, dv)], dim=2).reshape(N, L, 3 * h * d)
    assert torch.equal(dqkv, ref_dqkv)
    if bias is not None:
        assert torch.equal(db, db_ref)
    assert fwa._native.device_flags() == 0


@pytest.mark.parametrize("N,h,L,extras", [(48, 4, 144, True), (96, 3, 49, True), (16, 8, 144, False)])
def test_qkv_layout_matches_the_oracle(N, h, L, extras):
    # the fused layouts against the float64 oracle on the same quantised inputs (every window)
    import numpy as np

    d, dt = 32, torch.float16
    rng = fwa.Rng(N + h + L)
    qkv = fwa.fill_uniform(rng, (N, L, 3 * h * d), dtype=dt)
    do = fwa.fill_uniform(rng, (N, L, h * d), dtype=dt)
    bias = fwa.fill_uniform(rng, (h, L, L), -2.0, 2.0) if extras else None
    mask = torch.where(fwa.fill_uniform(rng, (4, L, L)) > 0.5, -100.0, 0.0).float().contiguous() \
        if extras else None
    sc = d ** -0.5
    assert fwa._native.launch_count() >= 0
    o = ops.attention_forward_qkv(qkv, h, sc, bias, mask, kernel="tc")
    dqkv, db = ops.attention_backward_qkv(qkv, do, h, sc, bias, mask, kernel="tc",
                                          want_dbias=extras)
    q5 = qkv.view(N, L, 3, h, d).double().cpu().numpy().transpose(2, 0, 3, 1, 4)   # (3, N, h, L, d)
    do4 = do.view(N, L, h, d).double().cpu().numpy().transpose(0, 2, 1, 3)
    bh = None if bias is None else bias.double().cpu().numpy()
    mh = None if mask is None else mask.double().cpu().numpy()
    ref_o, p = orc.attention_forward(q5[0], q5[1], q5[2], sc, bias=bh, mask=mh)
    grads = orc.attention_backward(q5[0], q5[1], q5[2], p, do4, sc, want_dbias=extras)
    got_o = o.view(N, L, h, d).double().cpu().numpy().transpose(0, 2, 1, 3)
    assert np.abs(got_o - ref_o).max() <= 2e-2
    g5 = dqkv.view(N, L, 3, h, d).double().cpu().numpy().transpose(2, 0, 3, 1, 4)
    for i in range(3):
        assert np.abs(g5[i] - grads[i]).max() <= 2e-2
    if extras:
        ref_db = grads[3]
        assert np.abs(db.double().cpu().numpy() - ref_db).max() <= 2e-2 * max(1.0, np.abs(ref_db).max())


def test_qkv_layout_falls_back_for_unsupported_shapes():
    rng = fwa.Rng(2)
    qkv = fwa.fill_uniform(rng, (6, 100, 3 * 2 * 24), dtype=torch.float16)  # L=100, d=24
    o = ops.attention_forward_qkv(qkv, 2, 0.2)
    ref, _ = _split_merge_reference(qkv, 2, 0.2, None, None)
    assert torch.equal(o, ref)
    with pytest.raises(fwa.CapacityError):
        ops.attention_forward_qkv(qkv, 2, 0.2, kernel="tc")


class SwinWindowAttentionRef(torch.nn.Module):
    """Plain fp32 torch (S)W-MSA block: the pattern the fused kernels replace."""

    def __init__(self, dim, heads, k, shift, qkv, proj, table):
        super().__init__()
        self.dim, self.h, self.k, self.shift = dim, heads, k, shift
        self.qkv, self.proj, self.table = qkv, proj, table

    def forward(self, x, mask):
        B, H, W, C = x.shape
        k, s, h = self.k, self.shift, self.h
        if s:
            x = torch.roll(x, (-s, -s), (1, 2))
        xw = x.view(B, H // k, k, W // k, k, C).permute(0, 1, 3, 2, 4, 5).reshape(-1, k * k, C)
        N, L, _ = xw.shape
        qkv = self.qkv(xw).view(N, L, 3, h, C // h).permute(2, 0, 3, 1, 4)
        q, kk, v = qkv[0], qkv[1], qkv[2]
        idx = torch.from_numpy(orc.relative_position_index(k)).cuda()
        bias = self.table[idx.view(-1)].view(L, L, h).permute(2, 0, 1)
        a = (q @ kk.transpose(-1, -2)) * (C // h) ** -0.5 + bias[None]
        if mask is not None:
            a = a + mask[torch.arange(N, device=x.device) % mask.shape[0]][:, None]
        o = (torch.softmax(a, -1) @ v).transpose(1, 2).reshape(N, L, C)
        y = self.proj(o).view(B, H // k, W // k, k, k, C).permute(0, 1, 3, 2, 4, 5).reshape(B, H, W, C)
        if s:
            y = torch.roll(y, (s, s), (1, 2))
        return y


@pytest.mark.parametrize("shift", [0, 3])
def test_swin_block_end_to_end_matches_torch(shift):
    torch.manual_seed(0)
    B, H, W, C, heads, k = 4, 28, 28, 96, 3, 7
    qkv_lin = torch.nn.Linear(C, 3 * C).cuda()
    proj = torch.nn.Linear(C, C).cuda()
    table = torch.nn.Parameter(0.02 * torch.randn((2 * k - 1) ** 2, heads, device="cuda"))
    x = torch.randn(B, H, W, C, device="cuda", requires_grad=True)
    mask = ops.shift_mask(H, W, k, shift) if shift else None

    # reference in fp32
    ref = SwinWindowAttentionRef(C, heads, k, shift, qkv_lin, proj, table)
    y_ref = ref(x, mask)
    g = torch.randn_like(y_ref)
    (y_ref * g).sum().backward()
    grads_ref = [t.grad.clone() for t in (x, qkv_lin.weight, proj.weight, table)]
    for t in (x, qkv_lin.weight, proj.weight, table):
        t.grad = None

    # fused path: bf16 attention through the package, autocast-free explicit casts
    xw = fwa.partition_windows(x, k, shift)
    qkv = qkv_lin(xw).to(torch.bfloat16).contiguous()
    bias = fwa.relative_position_bias(table, k)
    o = fwa.window_attention_qkv(qkv, heads, None, bias, mask)
    y = fwa.reverse_windows(proj(o.float()), k, H, W, shift)
    (y * g).sum().backward()
    dx = x.grad
    assert (y - y_ref).abs().max().item() <= 3e-2 * y_ref.abs().max().item()
    for got, want in zip((dx, qkv_lin.weight.grad, proj.weight.grad, table.grad), grads_ref):
        assert (got - want).abs().max().item() <= 3e-2 * max(1e-3, want.abs().max().item())


@pytest.mark.parametrize("shift", [0, 6])
def test_swin_b_block_window12_matches_torch(shift):
    """Swin-B geometry (window 12, L = 144, d = 32): the flat-row kernels with bias/mask/dBias."""
    torch.manual_seed(1)
    B, H, W, C, heads, k = 2, 24, 24, 128, 4, 12
    qkv_lin = torch.nn.Linear(C, 3 * C).cuda()
    proj = torch.nn.Linear(C, C).cuda()
    table = torch.nn.Parameter(0.02 * torch.randn((2 * k - 1) ** 2, heads, device="cuda"))
    x = torch.randn(B, H, W, C, device="cuda", requires_grad=True)
    mask = ops.shift_mask(H, W, k, shift) if shift else None

    ref = SwinWindowAttentionRef(C, heads, k, shift, qkv_lin, proj, table)
    y_ref = ref(x, mask)
    g = torch.randn_like(y_ref)
    (y_ref * g).sum().backward()
    grads_ref = [t.grad.clone() for t in (x, qkv_lin.weight, proj.weight, table)]
    for t in (x, qkv_lin.weight, proj.weight, table):
        t.grad = None

    xw = fwa.partition_windows(x, k, shift)
    qkv = qkv_lin(xw).to(torch.bfloat16).contiguous()
    bias = fwa.relative_position_bias(table, k)
    o = fwa.window_attention_qkv(qkv, heads, None, bias, mask)
    y = fwa.reverse_windows(proj(o.float()), k, H, W, shift)
    (y * g).sum().backward()
    assert (y - y_ref).abs().max().item() <= 3e-2 * y_ref.abs().max().item()
    for got, want in zip((x.grad, qkv_lin.weight.grad, proj.weight.grad, table.grad), grads_ref):
        assert (got - want).abs().max().item() <= 3e-2 * max(1e-3, want.abs().max().item())


@pytest.mark.parametrize("B,H,C,heads,k,shift", [(4, 28, 96, 3, 7, 3), (2, 24, 128, 4, 12, 6),
                                                 (2, 14, 384, 12, 7, 0)])
def test_swin_block_module_matches_torch_block(B, H, C, heads, k, shift):
    # fwa.SwinWindowAttention (kernels end to end) vs TorchSwinWindowAttention (plain torch
    # ops, same weights), bf16, forward and backward
    torch.manual_seed(1)
    blk = fwa.SwinWindowAttention(C, heads, k, shift)
    ref = fwa.TorchSwinWindowAttention(blk)
    x = torch.randn(B, H, H, C, device="cuda", dtype=torch.bfloat16)
    g = torch.randn_like(x)
    outs = []
    for m in (blk, ref):
        xr = x.clone().requires_grad_(True)
        y = m(xr)
        y.backward(g)
        outs.append((y.float(), xr.grad.float(), blk.qkv.weight.grad.float().clone(),
                     blk.table.grad.float().clone()))
        for t in (blk.qkv.weight, blk.qkv.bias, blk.proj.weight, blk.proj.bias, blk.table):
            t.grad = None
    for a, b in zip(*outs):
        tol = 3e-2 * max(1.0, b.abs().max().item())
        assert (a - b).abs().max().item() <= tol
