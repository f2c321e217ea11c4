"""Phase timeline of CTA 0 in the flat backward kernel (needs tools/micro/libfwa_trace.so).

python tools/micro/bflat_trace.py --shape 4096,4,144,32
"""
import argparse, ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
os.environ["FWA_LIB_PATH"] = os.environ.get("FWA_TRACE_LIB") or os.path.join(os.path.dirname(__file__), "libfwa_trace.so")
import paper_2501_06480_b200 as fwa
from paper_2501_06480_b200 import ops, _native

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096,4,144,32")
a = ap.parse_args()
N, h, L, d = map(int, a.shape.split(","))
rng = fwa.Rng(1)
q, k, v, do = (fwa.fill_uniform(rng, (N, h, L, d), dtype=torch.float16) for _ in range(4))
for _ in range(3):
    ops.attention_backward(q, k, v, do, d ** -0.5)
torch.cuda.synchronize()
lib = _native.load()
buf = (ctypes.c_longlong * (16 * 64))()
assert lib.fwa_bflat_trace_copy(buf) == 0
t = np.array(buf, dtype=np.int64).reshape(16, 64)
t0 = t[0, 0]
names = ["SdP_iss", "grad_beg", "grad_end", "sm_start", "p_stored", "p_ready", "ds_ready", "dq_out", "dV_done", "dK0_done", "dQ_done", "accw_beg", "accw_end", "dK1_done", "tc_done"]
print("blk " + " ".join(f"{n:>9}" for n in names))
for b in range(30):
    print(f"{b:3d} " + " ".join(f"{(t[e, b] - t0) if t[e, b] else -1:9d}" for e in range(15)))
