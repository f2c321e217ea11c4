"""Per-call device times of single window-attention layer calls (A/B of kernel builds).

Run from a repo root (this tree, or an older tree for a same-box A/B):
  python tools/time_layers.py [case ...]
Each case is timed as the average of 20 back-to-back launches (CUDA events on torch's
current stream) after 3 warm-up calls; inputs are > 2x L2, so every launch streams from HBM.
"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())

import torch  # noqa: E402

import paper_2501_06480_b200 as fwa  # noqa: E402
from paper_2501_06480_b200 import ops  # noqa: E402


def timed_graph(fn, reps=20):
    """Device us per call with `reps` calls captured in one CUDA graph (no host overhead)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def timed(fn, reps=20):
    """(device us per call, host us per call): host >= device means the loop is launch-bound."""
    import time

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    host = (time.perf_counter() - t0) / reps * 1e6
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3, host


def window_case(name, shape, dt, k, shift, reverse):
    B, H, W, C = shape
    x = fwa.fill_uniform(fwa.Rng(3), shape, dtype=dt)
    y = ops.window_partition(x, k, shift)
    fn = (lambda: ops.window_reverse(y, k, H, W, shift)) if reverse \
        else (lambda: ops.window_partition(x, k, shift))
    us, host = timed(fn)
    byts = 2 * x.numel() * x.element_size()
    return {"case": name, "us": round(us, 1), "GB/s": round(byts / us / 1e3), "host_us": round(host, 1)}


def case(name, shape, dt, bwd, bias, mask_nw, dbias, tokens=False):
    N, h, L, d = shape
    rng = fwa.Rng(7)
    q, k, v, do = (fwa.fill_uniform(rng, shape, dtype=dt) for _ in range(4))
    b = fwa.fill_uniform(rng, (h, L, L), -2.0, 2.0) if bias else None
    m = torch.where(fwa.fill_uniform(rng, (mask_nw, L, L)) > 0.5, -100.0, 0.0).float().contiguous() \
        if mask_nw else None
    sc = d ** -0.5
    if tokens:
        qkv = fwa.fill_uniform(rng, (N, L, 3 * h * d), dtype=dt)
        dO = fwa.fill_uniform(rng, (N, L, h * d), dtype=dt)
        fn = (lambda: ops.attention_backward_qkv(qkv, dO, h, sc, b, m, want_dbias=dbias)) if bwd \
            else (lambda: ops.attention_forward_qkv(qkv, h, sc, b, m))
    else:
        fn = (lambda: ops.attention_backward(q, k, v, do, sc, b, m, want_dbias=dbias)) if bwd \
            else (lambda: ops.attention_forward(q, k, v, sc, b, m))
    us, host = timed(fn)
    byts = (7 if bwd else 4) * N * h * L * d * 2
    return {"case": name, "us": round(us, 1), "GB/s": round(byts / us / 1e3), "host_us": round(host, 1)}


B1 = (4096, 4, 144, 32)
B3 = (256, 16, 144, 32)
B4 = (64, 32, 144, 32)
CASES = {
    "fwd": (B1, torch.float16, False, False, 0, False),
    "fwd_bias": (B1, torch.bfloat16, False, True, 0, False),
    "fwd_bias_mask": (B1, torch.bfloat16, False, True, 64, False),
    "fwd_bias_s3": (B3, torch.bfloat16, False, True, 4, False),
    "bwd": (B1, torch.float16, True, False, 0, False),
    "bwd_dbias": (B1, torch.bfloat16, True, True, 0, True),
    "bwd_bias": (B1, torch.bfloat16, True, True, 0, False),
    "bwd_bf16": (B1, torch.bfloat16, True, False, 0, False),
    "bwd_dbias_mask": (B1, torch.bfloat16, True, True, 64, True),
    "bwd_dbias_s2": ((1024, 8, 144, 32), torch.bfloat16, True, True, 16, True),
    "bwd_dbias_s3": (B3, torch.bfloat16, True, True, 4, True),
    "bwd_bias_s3": (B3, torch.bfloat16, True, True, 4, False),
    "bwd_s3": (B3, torch.bfloat16, True, False, 0, False),
    "bwd_dbias_s4": (B4, torch.bfloat16, True, True, 0, True),
    "fwd_tok": (B1, torch.float16, False, False, 0, False, True),
    "bwd_tok": (B1, torch.float16, True, False, 0, False, True),
    "bwd_tok_dbias": (B1, torch.bfloat16, True, True, 0, True, True),
    "t1_tok": ((8192, 3, 49, 32), torch.float16, False, False, 0, False, True),
    "t1_tok_bwd": ((8192, 3, 49, 32), torch.float16, True, False, 0, False, True),
}

# Swin-T stage layers, fwd fp16, timed inside a CUDA graph (the small ones are launch-bound
# eagerly); each call on its own rotating buffers so consecutive calls do not hit in L2
GRAPH_CASES = {"t0": (2, 3, 49, 32), "t00": (296, 3, 49, 32), "t1": (8192, 3, 49, 32), "t2": (2048, 6, 49, 32), "t3": (512, 12, 49, 32),
               "t4": (128, 24, 49, 32), "b1": (4096, 4, 144, 32), "b3": (256, 16, 144, 32),
               "l1": (61035, 1, 64, 32), "l2": (30517, 1, 64, 64), "l3": (15258, 1, 256, 32),
               "l4": (7629, 1, 256, 64)}


def graph_case(name, shape, bwd=False):
    N, h, L, d = shape
    rng = fwa.Rng(9)
    nbuf = max(2, int(2 * 126e6 // (4 * N * h * L * d * 2)) + 1)
    bufs = [tuple(fwa.fill_uniform(rng, shape, dtype=torch.float16) for _ in range(4)) for _ in range(nbuf)]
    outs = [torch.empty_like(b[0]) for b in bufs]
    it = [0]

    def fn():
        i = it[0] % nbuf
        it[0] += 1
        q, k, v, do = bufs[i]
        if bwd:
            ops.attention_backward(q, k, v, do, d ** -0.5)
        else:
            ops.attention_forward(q, k, v, d ** -0.5, out=outs[i])
    us = timed_graph(fn, reps=6 * nbuf)
    byts = (7 if bwd else 4) * N * h * L * d * 2
    return {"case": name + ("_bwd" if bwd else ""), "us": round(us, 2), "GB/s": round(byts / us / 1e3),
            "buffers": nbuf}


WINDOW_CASES = {
    "partition": ((128, 56, 56, 96), torch.bfloat16, 7, 3, False),
    "reverse": ((128, 56, 56, 96), torch.bfloat16, 7, 3, True),
    "partition_b": ((64, 96, 96, 128), torch.bfloat16, 12, 6, False),
    "reverse_b": ((64, 96, 96, 128), torch.bfloat16, 12, 6, True),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        if n.split("_")[0] in GRAPH_CASES:
            print(json.dumps(graph_case(n.split("_")[0], GRAPH_CASES[n.split("_")[0]], n.endswith("_bwd"))), flush=True)
        elif n in WINDOW_CASES:
            print(json.dumps(window_case(n, *WINDOW_CASES[n])), flush=True)
        else:
            print(json.dumps(case(n, *CASES[n])), flush=True)
