"""Swin-T stage-1 attention glue: split path (permute qkv, attention, permute O) vs fused qkv layout."""
import sys, json
import torch
sys.path.insert(0, ".")
import paper_2501_06480_b200 as fwa
from paper_2501_06480_b200 import ops

N, h, L, d = 8192, 3, 49, 32
rng = fwa.Rng(1)
qkv = fwa.fill_uniform(rng, (N, L, 3 * h * d), dtype=torch.float16)
sc = d ** -0.5

def split():
    q, k, v = (qkv.view(N, L, 3, h, d)[:, :, i].permute(0, 2, 1, 3).contiguous() for i in range(3))
    o = ops.attention_forward(q, k, v, sc)
    return o.permute(0, 2, 1, 3).reshape(N, L, h * d).contiguous()

def fused():
    return ops.attention_forward_qkv(qkv, h, sc)

res = {}
for name, fn in (("split", split), ("fused", fused)):
    for _ in range(3): fn()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / 10
print(json.dumps({"shape": [N, h, L, d], "ms_split_path": res["split"], "ms_fused_qkv": res["fused"],
                  "speedup": res["split"] / res["fused"]}))
