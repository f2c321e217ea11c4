"""dBias error of the flat backward's per-CTA partials (fp32 vs f16, FWA_DBIAS_PARTS) at
Swin-B stage shapes, against an fp32 torch autograd reference on the same inputs.

  python tools/dbias_precision.py            # prints one JSON line per (shape, dtype)

Run it once per FWA_DBIAS_PARTS setting (the choice is read once per process)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_06480_b200 as fwa  # noqa: E402
from paper_2501_06480_b200 import ops  # noqa: E402

SHAPES = [(4096, 4, 144, 32), (1024, 8, 144, 32), (256, 16, 144, 32)]


def ref_dbias(q, k, v, do, scale, bias, chunk=256):
    db = torch.zeros_like(bias)
    for n0 in range(0, q.shape[0], chunk):
        sl = slice(n0, n0 + chunk)
        qf, kf, vf = (t[sl].float().requires_grad_(True) for t in (q, k, v))
        bf = bias.clone().requires_grad_(True)
        s = (qf @ kf.transpose(-1, -2)) * scale + bf[None]
        (torch.softmax(s, -1) @ vf).backward(do[sl].float())
        db += bf.grad
    return db


def main():
    parts = os.environ.get("FWA_DBIAS_PARTS", "auto")
    for shape in SHAPES:
        N, h, L, d = shape
        for dt in (torch.float16, torch.bfloat16):
            rng = fwa.Rng(31 + N)
            q, k, v, do = (fwa.fill_uniform(rng, shape, dtype=dt) for _ in range(4))
            bias = fwa.fill_uniform(rng, (h, L, L), -3.0, 3.0)
            scale = d ** -0.5
            db = ops.attention_backward(q, k, v, do, scale, bias, None, want_dbias=True)[3]
            ref = ref_dbias(q, k, v, do, scale, bias)
            err = (db - ref).abs()
            print(json.dumps({"parts": parts, "shape": shape, "dtype": str(dt).replace("torch.", ""),
                              "max_abs_err": err.max().item(), "ref_absmax": ref.abs().max().item(),
                              "rel_max": err.max().item() / ref.abs().max().item(),
                              "rel_rms": (err.pow(2).mean().sqrt() / ref.pow(2).mean().sqrt()).item()}),
                  flush=True)


if __name__ == "__main__":
    main()
