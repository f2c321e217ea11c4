"""Benchmark: window-attention windows/s and % of B200 HBM roofline (BASELINE.json metric).

Default workload (BASELINE configs[1]): Swin-T at 224^2, B=128 images per GPU,
fp16 forward of all 12 window-attention layers (depths 2/2/6/2):
  stage 1 (8192, 3, 49, 32) x2, stage 2 (2048, 6, 49, 32) x2,
  stage 3 (512, 12, 49, 32) x6, stage 4 (128, 24, 49, 32) x2   [(N, h, L, d)]
One "step" = those 12 forward calls, each on its own resident Q/K/V (1.46 GB
of algorithmic traffic per step, > 10x the 126 MB L2, so no flush is needed).
value = windows processed per second over all ranks (window = all h heads).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fwa|reference]
                  [--workload swin_t_fwd|swin_t_fwdbwd|swin_b_fwdbwd]

Multi-GPU: torchrun, one process per GPU, weak scaling (B=128 per rank), no
collective on the hot path; barrier + synchronize around the timed region,
time = max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SWIN_T = [(8192, 3, 49, 32)] * 2 + [(2048, 6, 49, 32)] * 2 + [(512, 12, 49, 32)] * 6 + \
         [(128, 24, 49, 32)] * 2  # B=128, 224^2, window 7
SWIN_B384 = [(4096, 4, 144, 32)] * 2 + [(1024, 8, 144, 32)] * 2 + [(256, 16, 144, 32)] * 18 + \
            [(64, 32, 144, 32)] * 2  # B=64, 384^2, window 12
WORKLOADS = {
    # name: (layers, images per rank, windows per image per stage-1, dtype, passes, mask/bias)
    "swin_t_fwd": dict(layers=SWIN_T, batch=128, dtype="float16", bwd=False, extras=False,
                       k=7, hw=56, desc="Swin-T 224^2 B=128, 12 layers, fp16 forward (configs[1])"),
    "swin_t_fwdbwd": dict(layers=SWIN_T, batch=128, dtype="bfloat16", bwd=True, extras=True,
                          k=7, hw=56, desc="Swin-T 224^2 B=128, shifted-window mask + rel-pos "
                                           "bias, bf16 forward+backward (configs[2])"),
    "swin_b_fwdbwd": dict(layers=SWIN_B384, batch=64, dtype="float16", bwd=True, extras=False,
                          k=12, hw=96, desc="Swin-B 384^2 window 12 B=64, fp16 forward+backward "
                                            "(configs[3])"),
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


# ---------------------------------------------------------------------------
# nvidia-smi clock sampler (runs during warm-up + timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU reference (oracle port of flash.py Alg. 1/2, float64) on host cores
# ---------------------------------------------------------------------------
def _cpu_worker(args):
    layers, batch, n_images, extras, bwd, seed = args
    import numpy as np

    from oracle import flashwin_oracle as orc

    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    rng = orc.Rng(seed)
    spent = 0.0
    windows = 0
    for (N, h, L, d) in layers:
        per_img = N // batch
        n = per_img * n_images
        q, kk, v = (orc.fill_uniform(rng, (n, h, L, d)) for _ in range(3))
        do = orc.fill_uniform(rng, (n, h, L, d)) if bwd else None
        r = max(1, d // 16)
        t0 = time.perf_counter()  # inputs are resident before timing, like the GPU arm
        orc.tiled_forward(q, kk, v, r, d ** -0.5)
        if bwd:
            orc.tiled_backward(q, kk, v, do, r, d ** -0.5)
        spent += time.perf_counter() - t0
        windows += n
    return windows, spent


def cpu_reference(wl, seconds_target=12.0, steps=1, warmup=0):
    """Time the oracle port on all host cores; returns windows/s (+ sample description)."""
    import multiprocessing as mp

    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    cores = len(os.sched_getaffinity(0))
    layers = wl["layers"]
    # calibrate: one image through all layers on one core
    w, t = _cpu_worker((layers, wl["batch"], 1, wl["extras"], wl["bwd"], 1))
    per_proc_images = max(1, int(seconds_target / max(t, 1e-3) / max(steps + warmup, 1)))
    ctx = mp.get_context("fork")
    results = []
    with ctx.Pool(cores) as pool:
        for s in range(warmup + steps):
            outs = pool.map(_cpu_worker, [(layers, wl["batch"], per_proc_images, wl["extras"],
                                           wl["bwd"], 100 + i) for i in range(cores)])
            dt = max(o[1] for o in outs)  # slowest process's compute time
            if s >= warmup:
                results.append((sum(o[0] for o in outs), dt))
    windows = sum(r[0] for r in results)
    secs = sum(r[1] for r in results)
    sample = (f"{per_proc_images} image(s) x {cores} processes per step through all "
              f"{len(layers)} layers, float64 oracle port of flash.py Alg.1"
              f"{'/2' if wl['bwd'] else ''} (numpy, 1 BLAS thread per process)")
    return windows / secs, cores, sample, secs / max(len(results), 1)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_gpu(args, wl):
    import torch
    import torch.distributed as dist

    import paper_2501_06480_b200 as fwa
    from paper_2501_06480_b200 import _native as nat
    from paper_2501_06480_b200 import ops

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    nat.load()
    dtype = getattr(torch, wl["dtype"])
    eb = torch.empty((), dtype=dtype).element_size()
    layers = wl["layers"]
    k = wl["k"]
    # per-rank inputs: every layer has its own resident Q/K/V(/dO)
    rng = fwa.Rng(42 + rank)
    bufs = []
    for (N, h, L, d) in layers:
        q, kk, v = (fwa.fill_uniform(rng, (N, h, L, d), dtype=dtype, device=dev) for _ in range(3))
        do = fwa.fill_uniform(rng, (N, h, L, d), dtype=dtype, device=dev) if wl["bwd"] else None
        bias = mask = None
        if wl["extras"]:
            table = fwa.fill_uniform(rng, ((2 * k - 1) ** 2, h), -0.04, 0.04, device=dev)
            bias = ops.bias_gather(table, k)
            # Swin alternates W-MSA / SW-MSA: the second block of each pair is shifted and
            # masked; the last stage (7x7 map = one window) never shifts.
            nW = N // wl["batch"]
            side = int(round(math.sqrt(nW))) * k
            idx_in_stage = sum(1 for x in layers[:len(bufs)] if x == (N, h, L, d))
            if nW > 1 and idx_in_stage % 2 == 1:
                mask = ops.shift_mask(side, side, k, k // 2, device=dev)
        o = torch.empty_like(q)
        bufs.append((q, kk, v, do, bias, mask, o, d ** -0.5))
    torch.cuda.synchronize()

    def step():
        for i, (q, kk, v, do, bias, mask, o, sc) in enumerate(bufs):
            ops.attention_forward(q, kk, v, sc, bias, mask, out=o)
            if wl["bwd"]:
                ops.attention_backward(q, kk, v, do, sc, bias, mask, want_dbias=bias is not None)

    sampler = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[0])
                           if os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")[0].isdigit()
                           else local)
    sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # One step = the 12 layer calls, captured once into a CUDA graph (launch-bound
    # small stages would otherwise measure Python/ctypes time, not the GPU).
    graph = None
    per_step_launches = None
    if not args.eager:
        graph = torch.cuda.CUDAGraph()
        l0 = nat.launch_count()
        with torch.cuda.graph(graph):
            step()
        per_step_launches = nat.launch_count() - l0
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
    # clock soak: keep the GPU busy ~1.5 s so nvidia-smi samples the loaded clocks
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < args.soak_s:
        for _ in range(20):
            graph.replay() if graph is not None else step()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = nat.launch_count()
    start.record()
    for s in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            step()
    stop.record()
    torch.cuda.synchronize()
    launches = nat.launch_count() - launches0
    if graph is not None:
        launches = per_step_launches * args.steps
    elapsed_ms = start.elapsed_time(stop)
    if world > 1:
        t = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
        dist.barrier()
    clocks = sampler.stop()

    # Per-layer kernel durations (roofline numerator): each distinct layer shape
    # replayed R times inside its own graph, CUDA events around the replays.
    reps = 10
    per_shape = {}
    for i, lay in enumerate(layers):
        if lay in per_shape:
            continue
        q, kk, v, do, bias, mask, o, sc = bufs[i]
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1):
            for _ in range(reps):
                ops.attention_forward(q, kk, v, sc, bias, mask, out=o)
                if wl["bwd"]:
                    ops.attention_backward(q, kk, v, do, sc, bias, mask, want_dbias=bias is not None)
        g1.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g1.replay()
        e1.record()
        torch.cuda.synchronize()
        per_shape[lay] = e0.elapsed_time(e1) / reps
        del g1
    per_layer_ms = [per_shape[lay] for lay in layers]
    windows_per_step = sum(N for (N, h, L, d) in layers)
    fwd_bytes = [4 * N * h * L * d * eb for (N, h, L, d) in layers]
    bwd_bytes = [7 * N * h * L * d * eb for (N, h, L, d) in layers] if wl["bwd"] else [0] * len(layers)
    alg_bytes_step = sum(fwd_bytes) + sum(bwd_bytes)
    flops_step = sum(4 * N * h * L * L * d for (N, h, L, d) in layers) + \
        (sum(10 * N * h * L * L * d for (N, h, L, d) in layers) if wl["bwd"] else 0)
    ms_per_step = elapsed_ms / args.steps
    value = windows_per_step * world / (ms_per_step / 1e3)
    peak, peak_src = load_peaks()
    kernel_ms = sum(per_layer_ms)
    achieved = alg_bytes_step / (kernel_ms / 1e3) / 1e9
    # dominant launch: the stage-1 layers (largest units count)
    dom = max(range(len(layers)), key=lambda i: fwd_bytes[i] + bwd_bytes[i])
    dom_gbs = (fwd_bytes[dom] + bwd_bytes[dom]) / (per_layer_ms[dom] / 1e3) / 1e9
    fp = ops.footprint(*layers[0], dtype=dtype)

    # ---- e2e through the public API with pinned host buffers --------------
    e2e = None
    if not args.no_e2e:
        host = []
        for (q, kk, v, do, bias, mask, o, sc) in bufs:
            host.append(tuple(t.cpu().pin_memory() if t is not None else None for t in (q, kk, v, do)))
        cfg_r = max(1, layers[0][3] // 16)

        def e2e_step():
            res = []
            for (qh, kh, vh, doh), (_, _, _, _, bias, mask, _, sc) in zip(host, bufs):
                cfg = fwa.TileConfig(r=cfg_r, scale=sc)
                o, ctx, _ = fwa.batched_flash_forward(qh, kh, vh, cfg, [fwa.ScratchpadArena(1 << 20)],
                                                      bias=bias, mask=mask)
                res.append(o)
                if wl["bwd"]:
                    res.extend(fwa.batched_flash_backward(ctx, doh, [fwa.ScratchpadArena(1 << 20)])[:3])
            return res
        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        if world > 1:
            t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        n_in = 4 if wl["bwd"] else 3
        n_out = 4 if wl["bwd"] else 1
        per_layer = [N * h * L * d * eb for (N, h, L, d) in layers]
        e2e = {"value": windows_per_step * world / e2e_s, "unit": "windows/s",
               "h2d_bytes_per_step": n_in * sum(per_layer), "d2h_bytes_per_step": n_out * sum(per_layer),
               "path": "paper_2501_06480_b200.batched_flash_forward"
                       f"{'/batched_flash_backward' if wl['bwd'] else ''} on pinned host torch "
                       "tensors (H2D copy + kernels + D2H of the outputs)",
               "steps": e2e_steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v_cpu, cores, sample, _ = cpu_reference(wl, seconds_target=args.cpu_seconds)
        cpu = {"value": v_cpu, "unit": "windows/s", "cores": cores, "kind": "port", "sample": sample}

    if rank == 0:
        line = {
            "metric": "window-attn windows/s (Swin-T B=128 fp16 fwd, 12 layers)"
            if args.workload == "swin_t_fwd" else f"window-attn windows/s ({wl['desc']})",
            "value": value, "unit": "windows/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": {"float16": "f16", "bfloat16": "bf16"}[wl["dtype"]],
            "data": "synthetic (SplitMix64 U[-1,1), seed 42+rank)",
            "config": {"workload": args.workload, "desc": wl["desc"], "images_per_gpu": wl["batch"],
                       "layers": [list(x) for x in layers], "global_batch": wl["batch"] * world,
                       "parallelism": f"dp{world} (weak: {wl['batch']} images per GPU, no collective)",
                       "launch": "eager" if args.eager else "CUDA graph of one step (12 layer calls), PDL between kernels",
                       "l2": "no flush: each step streams "
                             f"{alg_bytes_step / 1e9:.2f} GB of distinct tensors (>> 126 MB L2)"},
            "tflops": flops_step * world / (ms_per_step / 1e3) / 1e12,
            "hbm_frac_step": alg_bytes_step / (ms_per_step / 1e3) / 1e9 / peak,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                         "kernel": f"fwa_{'fwd+bwd' if wl['bwd'] else 'fwd'} ({fp['kernel_fwd']})",
                         "algorithmic_bytes_per_step": alg_bytes_step,
                         "dominant_launch": {"shape": list(layers[dom]), "ms": per_layer_ms[dom],
                                             "GB/s": dom_gbs, "frac": dom_gbs / peak},
                         "per_layer_ms": per_layer_ms,
                         "how": "per-launch time = CUDA events around a graph of 10 back-to-back "
                                "launches of that layer; achieved = algorithmic bytes / sum of "
                                "per-layer launch times"},
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clocks,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_reference(args, wl):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    v, cores, sample, per_step = cpu_reference(wl, seconds_target=args.cpu_seconds,
                                               steps=args.steps, warmup=args.warmup)
    line = {
        "impl": "reference",
        "metric": "window-attn windows/s (Swin-T B=128 fp16 fwd, 12 layers)"
        if args.workload == "swin_t_fwd" else f"window-attn windows/s ({wl['desc']})",
        "value": v, "unit": "windows/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SplitMix64 U[-1,1))",
        "config": {"workload": args.workload, "desc": wl["desc"],
                   "note": "reference CPU path = oracle port (oracle/flashwin_oracle.py) of "
                           "flash.py Alg.1/2 in float64 on all host cores; the reference itself is "
                           "pure Python and is not shipped to the GPU box"},
        "cpu_baseline": {"value": v, "unit": "windows/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "windows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="fwa", choices=["fwa", "reference"])
    ap.add_argument("--workload", default="swin_t_fwd", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--eager", action="store_true", help="no CUDA graph for the timed steps")
    ap.add_argument("--soak-s", type=float, default=1.5, help="loaded seconds before timing (clock sampling)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_gpu(args, wl)


if __name__ == "__main__":
    main()
