"""Raw CTA-0 event table of the flat backward trace build (events 0..15, relative to event 0 of block 0)."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
os.environ["FWA_LIB_PATH"] = os.environ.get("FWA_TRACE_LIB") or os.path.join(os.path.dirname(__file__), "libfwa_trace.so")
import paper_2501_06480_b200 as fwa
from paper_2501_06480_b200 import ops, _native
N, h, L, d = 4096, 4, 144, 32
rng = fwa.Rng(1)
q, k, v, do = (fwa.fill_uniform(rng, (N, h, L, d), dtype=torch.float16) for _ in range(4))
ops.attention_backward(q, k, v, do, d ** -0.5)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (16 * 64))()
assert _native.load().fwa_bflat_trace_copy(buf) == 0
t = np.array(buf, dtype=np.int64).reshape(16, 64)
t0 = t[0, 0]
ev = [int(x) for x in sys.argv[1:]] or list(range(16))
print("blk " + " ".join(f"{e:>7d}" for e in ev))
for b in range(1, 9):
    print(f"{b:3d} " + " ".join(f"{(t[e, b] - t0) if t[e, b] else -1:7d}" for e in ev))
