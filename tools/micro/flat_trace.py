"""Phase timeline of CTA 0 in the flat forward kernel (needs tools/micro/libfwa_trace.so).

python tools/micro/flat_trace.py --shape 4096,4,144,32
"""
import argparse, ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_2501_06480_b200 import _native
_native.LIB_PATH = os.path.join(os.path.dirname(__file__), "libfwa_trace.so")
import paper_2501_06480_b200 as fwa
from paper_2501_06480_b200 import ops

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096,4,144,32")
a = ap.parse_args()
N, h, L, d = map(int, a.shape.split(","))
rng = fwa.Rng(1)
q, k, v = (fwa.fill_uniform(rng, (N, h, L, d), dtype=torch.float16) for _ in range(3))
for _ in range(3):
    o = ops.attention_forward(q, k, v, d ** -0.5)
torch.cuda.synchronize()
lib = _native.load()
buf = (ctypes.c_longlong * (8 * 64))()
assert lib.fwa_flat_trace_copy(buf) == 0
t = np.array(buf, dtype=np.int64).reshape(8, 64)
t0 = t[0, 0]
names = ["S_wait0", "S_issue", "PV_issue", "sm_start", "sm_end", "o_full", "epi_end"]
print("blk " + " ".join(f"{n:>9}" for n in names))
for b in range(40):
    print(f"{b:3d} " + " ".join(f"{(t[e, b] - t0) if t[e, b] else -1:9d}" for e in range(7)))
