import sys, torch
sys.path.insert(0, ".")
import paper_2501_06480_b200 as fwa
ops = fwa.ops
N, h, L, d = 64, 3, 49, 32
dt = torch.float16
rng = fwa.Rng(N * 7 + h)
qkv = fwa.fill_uniform(rng, (N, L, 3 * h * d), dtype=dt)
do = fwa.fill_uniform(rng, (N, L, h * d), dtype=dt)
bias = fwa.fill_uniform(rng, (h, L, L), -0.3, 0.3)
mask = torch.where(fwa.fill_uniform(rng, (4, L, L)) > 0.5, -100.0, 0.0).float().contiguous()
sc = d ** -0.5
for wd in (True, False):
    dqkv, db = ops.attention_backward_qkv(qkv, do, h, sc, bias, mask, want_dbias=wd)
    q, k, v = (qkv.view(N, L, 3, h, d)[:, :, i].permute(0, 2, 1, 3).contiguous() for i in range(3))
    do4 = do.view(N, L, h, d).permute(0, 2, 1, 3).contiguous()
    dq, dk, dv, dbr = ops.attention_backward(q, k, v, do4, sc, bias, mask, want_dbias=wd)
    ref = torch.stack([t.permute(0, 2, 1, 3) for t in (dq, dk, dv)], dim=2).reshape(N, L, 3 * h * d)
    diff = (dqkv.float() - ref.float()).abs().view(N, L, 3, h, d)
    print("want_dbias", wd, [diff[:, :, i].max().item() for i in range(3)], "neq count", (diff > 0).sum().item())
    print("nan qkv", torch.isnan(dqkv).sum().item(), "nan split", [torch.isnan(t).sum().item() for t in (dq, dk, dv)])
    bad = torch.isnan(dq).nonzero()[:5]
    print("first nan dq idx (n,h,row,col)", bad.tolist())
