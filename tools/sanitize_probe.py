"""Tiny run of every libfwa kernel family, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2501_06480_b200 as fwa
from paper_2501_06480_b200 import ops

rng = fwa.Rng(3)
for dt in (torch.float16, torch.bfloat16):
    for shape in [(5, 2, 49, 32), (3, 1, 64, 64), (4, 1, 36, 16), (3, 2, 144, 32), (2, 1, 256, 32)]:
        q, k, v, do = (fwa.fill_uniform(rng, shape, dtype=dt) for _ in range(4))
        o = ops.attention_forward(q, k, v, 0.3)
        dq, dk, dv, _ = ops.attention_backward(q, k, v, do, 0.3)
    N, h, L = 6, 2, 49
    q, k, v, do = (fwa.fill_uniform(rng, (N, h, L, 32), dtype=dt) for _ in range(4))
    bias = fwa.fill_uniform(rng, (h, L, L), -0.5, 0.5)
    mask = ops.shift_mask(14, 21, 7, 3)
    ops.attention_forward(q, k, v, 0.3, bias, mask)
    ops.attention_backward(q, k, v, do, 0.3, bias, mask, want_dbias=True)
q, k, v, do = (fwa.fill_uniform(rng, (3, 2, 20, 10)) for _ in range(4))
ops.attention_forward(q, k, v, 0.3)
ops.attention_backward(q, k, v, do, 0.3)
x = fwa.fill_uniform(rng, (1, 14, 14, 8), dtype=torch.float16)
ops.window_reverse(ops.window_partition(x, 7, 3), 7, 14, 14, 3)
torch.cuda.synchronize()
print("probe ok, device flags", fwa._native.device_flags())
