"""In-kernel MMA execution times of the flat backward (TC-only build with serializing probes).

FWA_TRACE_LIB=tools/micro/libfwa_tconly.so python tools/micro/bflat_probe.py
"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
os.environ["FWA_LIB_PATH"] = os.environ.get("FWA_TRACE_LIB") or os.path.join(os.path.dirname(__file__), "libfwa_tconly.so")
import paper_2501_06480_b200 as fwa
from paper_2501_06480_b200 import ops, _native

N, h, L, d = 4096, 4, 144, 32
rng = fwa.Rng(1)
q, k, v, do = (fwa.fill_uniform(rng, (N, h, L, d), dtype=torch.float16) for _ in range(4))
for _ in range(2):
    ops.attention_backward(q, k, v, do, d ** -0.5)
torch.cuda.synchronize()
lib = _native.load()
buf = (ctypes.c_longlong * (16 * 64))()
assert lib.fwa_bflat_trace_copy(buf) == 0
t = np.array(buf, dtype=np.int64).reshape(16, 64)
print("blk  SdP_issue->exec  dV(issue->exec)  dK0  dQ  dK1")
for b in range(2, 14):
    sdp = t[15, b] - t[0, b]
    dv = t[4, b] - t[1, b]
    dk0 = t[5, b] - t[4, b]
    dq = t[6, b] - t[5, b]
    dk1 = (t[7, b] - t[6, b]) if t[7, b] else -1
    print(f"{b:3d} {sdp:8d} {dv:8d} {dk0:8d} {dq:8d} {dk1:8d}")
