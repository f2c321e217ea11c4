"""Time the large-window backward (bwd only, L2 flushed) for a few (L, d) shapes.

python tools/time_bwd_large.py            # whatever kernel the library picks
FWA_NO_FLAT=1 python tools/time_bwd_large.py   # the pre-flat path, for comparison
Prints one line per shape: kernel, us per launch, algorithmic GB/s (7 L d s per unit).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_06480_b200 as fwa

ops = fwa.ops
shapes = [(8192, 256, 32), (8192, 208, 32), (8192, 144, 32), (16384, 96, 64), (16384, 112, 64),
          (8192, 256, 16)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1:]]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for units, L, d in shapes:
    rng = fwa.Rng(1)
    q, k, v, do = (fwa.fill_uniform(rng, (units, 1, L, d), dtype=torch.float16) for _ in range(4))
    fp = ops.footprint(units, 1, L, d, torch.float16)
    for _ in range(3):
        ops.attention_backward(q, k, v, do, d ** -0.5)
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ops.attention_backward(q, k, v, do, d ** -0.5)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    ms = ts[len(ts) // 2]
    gbs = 7 * L * d * 2 * units / (ms * 1e-3) / 1e9
    print(f"L={L} d={d} units={units} kernel_bwd={fp.get('kernel_bwd')} {ms * 1e3:.1f} us {gbs:.0f} GB/s "
          f"({gbs / 6450:.1%} of 6450)", flush=True)
