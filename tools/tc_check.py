"""Quick TC-kernel parity probe (developer tool): prints max errors vs a torch fp32 reference."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2501_06480_b200 as fwa
from paper_2501_06480_b200 import ops

torch.manual_seed(0)
for dt in (torch.float16, torch.bfloat16):
    for (N, h, L, d) in [(1, 2, 64, 32), (1, 1, 49, 32), (4, 3, 49, 32), (5, 3, 49, 32), (2, 2, 64, 64),
                         (3, 1, 16, 16), (700, 3, 49, 32), (8192, 3, 49, 32), (33, 5, 36, 64),
                         (64, 4, 144, 32), (100, 2, 256, 32), (37, 3, 256, 64), (50, 2, 100, 16), (33, 1, 81, 32), (4096, 4, 144, 32)]:
        q, k, v = (torch.rand(N, h, L, d, device="cuda", dtype=torch.float32).mul_(2).sub_(1).to(dt) for _ in range(3))
        sc = d ** -0.5
        ref = torch.softmax((q.float() @ k.float().transpose(-1, -2)) * sc, -1) @ v.float()
        try:
            o = ops.attention_forward(q, k, v, sc, kernel="tc")
            torch.cuda.synchronize()
            err = (o.float() - ref).abs().max().item()
            print(f"{dt} {(N,h,L,d)} tc err={err:.3e} {'OK' if err < 2e-2 else 'FAIL'}", flush=True)
        except Exception as e:
            print(f"{dt} {(N,h,L,d)} EXC {type(e).__name__}: {e}", flush=True)
