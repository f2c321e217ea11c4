"""Quick TC-backward parity probe (developer tool) vs torch fp32 autograd."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2501_06480_b200 as fwa
from paper_2501_06480_b200 import ops, _native

torch.manual_seed(0)
for dt in (torch.float16, torch.bfloat16):
    for (N, h, L, d) in [(1, 2, 64, 32), (1, 1, 49, 32), (4, 3, 49, 32), (5, 3, 49, 32), (2, 2, 64, 64),
                         (3, 1, 16, 16), (700, 3, 49, 32), (8192, 3, 49, 32), (33, 5, 36, 64),
                         (64, 4, 144, 32), (100, 2, 256, 32), (37, 3, 128, 64), (50, 2, 100, 16), (33, 1, 81, 32), (61, 2, 200, 16), (4096, 4, 144, 32)]:
        q, k, v, do = (torch.rand(N, h, L, d, device="cuda").mul_(2).sub_(1).to(dt) for _ in range(4))
        sc = d ** -0.5
        qf, kf, vf = (t.float().requires_grad_() for t in (q, k, v))
        o = torch.softmax((qf @ kf.transpose(-1, -2)) * sc, -1) @ vf
        o.backward(do.float())
        try:
            dq, dk, dv, _ = ops.attention_backward(q, k, v, do, sc, kernel="tc")
            torch.cuda.synchronize()
            errs = [(a.float() - b.grad).abs().max().item() for a, b in ((dq, qf), (dk, kf), (dv, vf))]
            ok = all(e < 2e-2 for e in errs)
            print(f"{dt} {(N,h,L,d)} dq/dk/dv err={errs[0]:.2e}/{errs[1]:.2e}/{errs[2]:.2e} {'OK' if ok else 'FAIL'}", flush=True)
        except Exception as e:
            print(f"{dt} {(N,h,L,d)} EXC {type(e).__name__}: {e}", flush=True)
print("device flags:", _native.device_flags())
