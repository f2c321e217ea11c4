"""Run one window-attention shape a few times (for ncu captures and quick timing).

python tools/profile_fwd.py --shape 8192,3,49,32 --dtype f16 --iters 5 [--bwd] [--kernel auto]
"""
import argparse, sys
import torch
sys.path.insert(0, ".")
import paper_2501_06480_b200 as fwa
from paper_2501_06480_b200 import ops

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="8192,3,49,32")
ap.add_argument("--dtype", default="f16")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--kernel", default="auto")
ap.add_argument("--bwd", action="store_true")
ap.add_argument("--extras", action="store_true")
a = ap.parse_args()
N, h, L, d = map(int, a.shape.split(","))
dt = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}[a.dtype]
rng = fwa.Rng(1)
q, k, v, do = (fwa.fill_uniform(rng, (N, h, L, d), dtype=dt) for _ in range(4))
bias = mask = None
if a.extras:
    kw = int(round(L ** 0.5))
    bias = ops.bias_gather(fwa.fill_uniform(rng, ((2 * kw - 1) ** 2, h), -0.05, 0.05), kw)
    mask = ops.shift_mask(8 * kw, 8 * kw, kw, kw // 2)
o = torch.empty_like(q)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for i in range(a.iters):
    ev[0].record()
    ops.attention_forward(q, k, v, d ** -0.5, bias, mask, kernel=a.kernel, out=o)
    if a.bwd:
        ops.attention_backward(q, k, v, do, d ** -0.5, bias, mask, kernel=a.kernel, want_dbias=bias is not None)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
eb = q.element_size()
byt = (4 + (7 if a.bwd else 0)) * N * h * L * d * eb
best = min(ts[1:] if len(ts) > 1 else ts)
print(f"shape={a.shape} dtype={a.dtype} bwd={a.bwd} best_ms={best:.4f} GB/s={byt/best/1e6:.1f} "
      f"frac={byt/best/1e6/6450:.3f} kernel={ops.footprint(N,h,L,d,dt)}")
