"""Cost of the Swin extras in the large-window backward: plain vs bias+mask vs +dBias.

python tools/time_bwd_add.py [N h L]      (default Swin-B 384 stage 1: 4096 4 144, d = 32)
Times ops.attention_backward (L2 flushed before each launch; median of 10) in bf16.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2501_06480_b200 as fwa

ops = fwa.ops
N, h, L = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 4, 144)
d, dt = 32, torch.bfloat16
rng = fwa.Rng(1)
q, k, v, do = (fwa.fill_uniform(rng, (N, h, L, d), dtype=dt) for _ in range(4))
bias = fwa.fill_uniform(rng, (h, L, L), -0.5, 0.5)
win = int(round(L ** 0.5))
assert win * win == L, "square windows only"
mask = ops.shift_mask(8 * win, 8 * win, win, win // 2)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[5] * 1e3


s = d ** -0.5
for name, fn in [("plain", lambda: ops.attention_backward(q, k, v, do, s)),
                 ("bias+mask", lambda: ops.attention_backward(q, k, v, do, s, bias, mask)),
                 ("bias+mask+dBias", lambda: ops.attention_backward(q, k, v, do, s, bias, mask,
                                                                    want_dbias=True))]:
    print(f"N={N} h={h} L={L} {name}: {timed(fn):.1f} us", flush=True)
