"""Benchmark: window-attention windows/s and % of B200 HBM roofline (BASELINE.json metric).

Default workload (BASELINE configs[1]): Swin-T at 224^2, B=128 images per GPU,
fp16 forward of all 12 window-attention layers (depths 2/2/6/2):
  stage 1 (8192, 3, 49, 32) x2, stage 2 (2048, 6, 49, 32) x2,
  stage 3 (512, 12, 49, 32) x6, stage 4 (128, 24, 49, 32) x2   [(N, h, L, d)]
One "step" = those 12 forward calls, each on its own resident Q/K/V (1.46 GB
of algorithmic traffic per step, > 10x the 126 MB L2, so no flush is needed),
replayed from a CUDA graph. value = windows processed per second over all
ranks (a window = all h heads of one window).

The same line carries "fwd_bwd": BASELINE configs[2] (Swin-T B=128, bf16,
relative-position bias on every layer (learnable: dBias computed), shifted-window
mask on the SW-MSA layers, forward + backward) measured the same way.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fwa|reference]
                  [--workload swin_t_fwd|swin_t_fwdbwd|swin_b_fwdbwd|swin_b_train|large_sweep]

Multi-GPU: torchrun, one process per GPU, weak scaling (B images per rank), no
collective on the hot path; barrier + synchronize around the timed region,
time = max over ranks (all_reduce MAX).
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
LARGE = [(61035, 1, 64, 32), (30517, 1, 64, 64), (15258, 1, 256, 32), (7629, 1, 256, 64)]
WORKLOADS = {
    "swin_t_fwd": dict(layers=SWIN_T, batch=128, dtype="float16", bwd=False, extras=False, k=7,
                       desc="Swin-T 224^2 B=128, 12 layers, fp16 forward (configs[1])"),
    "swin_t_fwdbwd": dict(layers=SWIN_T, batch=128, dtype="bfloat16", bwd=True, extras=True, k=7,
                          desc="Swin-T 224^2 B=128, rel-pos bias (learnable) + shifted-window "
                               "mask on SW-MSA layers, bf16 forward+backward (configs[2])"),
    "swin_b_fwdbwd": dict(layers=SWIN_B384, batch=64, dtype="float16", bwd=True, extras=False,
                          k=12, desc="Swin-B 384^2 window 12 B=64, fp16 forward+backward "
                                     "(configs[3])"),
    "swin_b_train": dict(layers=SWIN_B384, batch=64, dtype="bfloat16", bwd=True, extras=True,
                         k=12, desc="Swin-B 384^2 window 12 B=64, rel-pos bias (learnable) + "
                                    "shifted-window mask on SW-MSA layers, bf16 forward+backward "
                                    "(configs[3] with configs[2]'s training extras)"),
    "large_sweep": dict(layers=LARGE, batch=1, cpu_div=512, dtype="float16", bwd=False, extras=False, k=8,
                        desc="large-window sweep L=64/256, d=32/64, ~1 GB per call, fp16 "
                             "forward (configs[4])"),
    "large_sweep_fwdbwd": dict(layers=LARGE[:3], batch=1, cpu_div=512, dtype="float16", bwd=True,
                               extras=False, k=8,
                               desc="large-window sweep fp16 forward+backward (configs[4]) on the "
                                    "shapes whose backward runs on tcgen05: L=64 d=32/64, L=256 "
                                    "d=32 (L=256 d=64 backward exceeds the flat kernel's TMEM/SMEM "
                                    "budget and runs on the SIMT kernel: DESIGN.md section 8)"),
}
METRIC = "window-attn windows/s + % HBM roofline"
# measured on the default run beside the headline (configs[2], [3] plain and with training
# extras, [4] forward and forward+backward)
EMBEDDED = ("swin_t_fwdbwd", "swin_b_fwdbwd", "swin_b_train", "large_sweep", "large_sweep_fwdbwd")
# (B, H, C, heads, window, shift): Swin-T 224^2 stage 1 (SW-MSA) and stage 3 (W-MSA) at B=128,
# Swin-B 384^2 window 12 stage 1 (SW-MSA) at B=64
BLOCKS = ((128, 56, 96, 3, 7, 3), (128, 14, 384, 12, 7, 0), (64, 96, 128, 4, 12, 6))


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def load_ncu_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# nvidia-smi clock sampler (runs during the clock soak + timed region)
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
# CPU reference on host cores: the stock reference package (baseline/_ref, installed
# from /root/reference/pkg) through its own public API, else the oracle port
# ---------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def ref_kind() -> str:
    return "reference" if os.path.isdir(os.path.join(REF_DIR, "flashwin")) else "port"


def _cpu_worker(args):
    layers, batch, n_images, bwd, seed, kind = args
    spent = 0.0
    windows = 0
    if kind == "reference":
        # the reference's own code path, as its harness times it (harness.py:537-559):
        # batched_flash_forward over the (B, h, L, C) stack, then flash_backward per slice
        sys.path.insert(0, REF_DIR)
        import flashwin as fw

        rng = fw.Rng(seed)
        for (N, h, L, d) in layers:
            n = max(1, N // batch) * n_images
            q, kk, v = (fw.fill_uniform(rng, (n, h, L, d), -1.0, 1.0) for _ in range(3))
            do = fw.fill_uniform(rng, (n, h, L, d), -1.0, 1.0) if bwd else None
            cfg = fw.TileConfig(r=max(1, d // 16), scale=d ** -0.5)
            arena = fw.ScratchpadArena(1 << 20)   # L = 144 backward needs > the 128 KB default
            t0 = time.perf_counter()  # inputs are resident before timing, like the GPU arm
            _, ctxs, _ = fw.batched_flash_forward(q, kk, v, cfg, [arena])
            if bwd:
                for b in range(n):
                    for hd in range(h):
                        fw.flash_backward(ctxs[b][hd], fw.DenseTensor((L, d), do.array[b, hd]), arena)
            spent += time.perf_counter() - t0
            windows += n
        return windows, spent
    from oracle import flashwin_oracle as orc

    rng = orc.Rng(seed)
    for (N, h, L, d) in layers:
        n = max(1, N // batch) * n_images
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
    """Time the reference CPU path on all host cores (one process per core, each on its own
    shard, inputs resident); returns (windows/s, cores, sample, s/step, kind)."""
    import multiprocessing as mp

    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    cores = len(os.sched_getaffinity(0))
    layers = wl["layers"]
    # one CPU sample "image" = N / cpu_div windows of every layer (cpu_div defaults to the
    # batch: one real image; the large sweep has no images, 1/512 of each ~1 GB call)
    div = wl.get("cpu_div", wl["batch"])
    kind = ref_kind()
    _, t = _cpu_worker((layers, div, 1, wl["bwd"], 1, kind))
    per_proc = max(1, int(seconds_target / max(t, 1e-3) / max(steps + warmup, 1)))
    results = []
    # spawn, not fork: the parent holds a CUDA context (forking it can hang the children)
    with mp.get_context("spawn").Pool(cores) as pool:
        for s in range(warmup + steps):
            outs = pool.map(_cpu_worker, [(layers, div, per_proc, wl["bwd"], 100 + i, kind)
                                          for i in range(cores)])
            if s >= warmup:
                results.append((sum(o[0] for o in outs), max(o[1] for o in outs)))
    windows = sum(r[0] for r in results)
    secs = sum(r[1] for r in results)
    unit = "image(s)" if div == wl["batch"] else f"1/{div}-of-call slice(s)"
    what = ("the stock reference flashwin (baseline/_ref) batched_flash_forward"
            + (" + per-slice flash_backward" if wl["bwd"] else "")
            + (" (the reference has no Swin bias / mask: computed without them)"
               if wl.get("extras") else "")
            if kind == "reference" else
            f"float64 oracle port of flash.py Alg.1{'/2' if wl['bwd'] else ''}")
    sample = (f"{per_proc} {unit} x {cores} processes per step through all {len(layers)} "
              f"layers, {what} (numpy float64, 1 BLAS thread per process; windows/s = windows / "
              f"slowest process time)")
    return windows / secs, cores, sample, secs / max(len(results), 1), kind


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
class GpuWorkload:
    def __init__(self, wl, dev, seed):
        import torch

        import paper_2501_06480_b200 as fwa
        from paper_2501_06480_b200 import ops

        self.wl, self.dev, self.ops = wl, dev, ops
        self.dtype = getattr(torch, wl["dtype"])
        self.eb = torch.empty((), dtype=self.dtype).element_size()
        layers, k = wl["layers"], wl["k"]
        rng = fwa.Rng(seed)
        self.bufs = []
        for (N, h, L, d) in layers:
            q, kk, v = (fwa.fill_uniform(rng, (N, h, L, d), dtype=self.dtype, device=dev)
                        for _ in range(3))
            do = fwa.fill_uniform(rng, (N, h, L, d), dtype=self.dtype, device=dev) \
                if wl["bwd"] else None
            bias = mask = None
            if wl["extras"]:
                table = fwa.fill_uniform(rng, ((2 * k - 1) ** 2, h), -0.04, 0.04, device=dev)
                bias = ops.bias_gather(table, k)
                # Swin alternates W-MSA / SW-MSA: the second block of each pair is shifted
                # and masked; the last stage (a single 7x7 window) never shifts.
                nW = N // wl["batch"]
                side = int(round(math.sqrt(nW))) * k
                idx_in_stage = sum(1 for x in layers[:len(self.bufs)] if x == (N, h, L, d))
                if nW > 1 and idx_in_stage % 2 == 1:
                    mask = ops.shift_mask(side, side, k, k // 2, device=dev)
            o = torch.empty_like(q)
            self.bufs.append((q, kk, v, do, bias, mask, o, d ** -0.5))
        torch.cuda.synchronize()

    def layer(self, i, fwd=True, bwd=None):
        """One layer call as the autograd Function runs it: for large windows with bias /
        mask the (bias + mask) score table is built once and shared by fwd and bwd."""
        q, kk, v, do, bias, mask, o, sc = self.bufs[i]
        bwd = self.wl["bwd"] if bwd is None else bwd
        table = self.ops.build_add_table(*q.shape, q.dtype, bias, mask) \
            if fwd and bwd and (bias is not None or mask is not None) else None
        if fwd:
            self.ops.attention_forward(q, kk, v, sc, bias, mask, out=o, add_table=table)
        if bwd:
            self.ops.attention_backward(q, kk, v, do, sc, bias, mask, want_dbias=bias is not None,
                                        add_table=table)

    def step(self):
        for i in range(len(self.bufs)):
            self.layer(i)

    def bytes_per_step(self):
        fwd = sum(4 * N * h * L * d * self.eb for (N, h, L, d) in self.wl["layers"])
        bwd = sum(7 * N * h * L * d * self.eb for (N, h, L, d) in self.wl["layers"]) \
            if self.wl["bwd"] else 0
        return fwd + bwd

    def flops_per_step(self):
        f = sum(4 * N * h * L * L * d for (N, h, L, d) in self.wl["layers"])
        if self.wl["bwd"]:
            f += sum(10 * N * h * L * L * d for (N, h, L, d) in self.wl["layers"])
        return f


def timed_graph(torch, nat, work, steps, warmup, eager, soak_s, world, dist):
    for _ in range(warmup):
        work.step()
    torch.cuda.synchronize()
    graph, per_step = None, None
    if not eager:
        graph = torch.cuda.CUDAGraph()
        l0 = nat.launch_count()
        with torch.cuda.graph(graph):
            work.step()
        per_step = nat.launch_count() - l0
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
    run = graph.replay if graph is not None else work.step
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < soak_s:
        for _ in range(10):
            run()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = nat.launch_count()
    start.record()
    for _ in range(steps):
        run()
    stop.record()
    torch.cuda.synchronize()
    launches = per_step * steps if graph is not None else nat.launch_count() - l0
    ms = start.elapsed_time(stop)
    if world > 1:
        ms = max_over_ranks(torch, dist, ms, work.dev)
        dist.barrier()
    del graph
    return ms / steps, launches


def max_over_ranks(torch, dist, x, dev):
    """MAX all-reduce of a scalar (NCCL on the device; gloo on the host for the CPU smoke test)."""
    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=dev if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def flushed_launch_ms(torch, work, i, fwd, bwd, reps=21):
    """Median device time of one layer launch with L2 flushed before it.

    The flush READS a 512 MB buffer (a sum), so L2 is refilled with clean lines:
    no dirty flush data is written back while the timed kernel runs.
    """
    flush = torch.ones(512 * 1024 * 1024 // 4, dtype=torch.float32, device=work.dev)
    times = []
    for _ in range(reps + 1):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        work.layer(i, fwd=fwd, bwd=bwd)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    del flush
    return statistics.median(times[1:])


def streamed_launch_ms(torch, work, i, fwd, bwd, reps=20):
    """Average device time of one layer launch over `reps` back-to-back launches.

    Only used when the layer's algorithmic traffic is > 2x the 126 MB L2: a streaming pass
    over that much data leaves nothing of the next pass's head in L2, so every launch is
    cold, and the per-launch event overhead (several us) is amortised over `reps`.
    """
    for _ in range(2):
        work.layer(i, fwd=fwd, bwd=bwd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        work.layer(i, fwd=fwd, bwd=bwd)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


L2_BYTES = 126 * 1024 * 1024


def measure_window_copies(dev, reps=20):
    """K3/K4 (window_partition / window_reverse with the Swin cyclic shift) at the stage-1
    feature maps of Swin-T 224^2 B=128 and Swin-B 384^2 B=64: bytes moved = read + write of
    the map; average of `reps` back-to-back launches (each > 2x L2 is not guaranteed here:
    the maps are 77 / 151 MB, so the copy partly hits L2 -- reported as measured)."""
    import torch

    import paper_2501_06480_b200 as fwa
    from paper_2501_06480_b200 import ops

    peak, _ = load_peaks()
    out = []
    for (shape, k, shift) in (((128, 56, 56, 96), 7, 3), ((64, 96, 96, 128), 12, 6)):
        x = fwa.fill_uniform(fwa.Rng(3), shape, dtype=torch.bfloat16, device=dev)
        y = ops.window_partition(x, k, shift)
        B, H, W, C = shape
        for name, fn in (("partition", lambda: ops.window_partition(x, k, shift, )),
                         ("reverse", lambda: ops.window_reverse(y, k, H, W, shift))):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            byts = 2 * x.numel() * x.element_size()
            out.append({"op": name, "shape": list(shape), "window": k, "shift": shift,
                        "dtype": "bf16", "ms": ms, "GB/s": byts / ms / 1e6,
                        "frac": byts / ms / 1e6 / peak, "bytes": byts})
        del x, y
    return out


def shard_workload(wl, rank, world):
    """Strong scaling: this rank's contiguous range of the workload's fixed global batch
    (shard.shard_images: whole images, so window n keeps its mask index n mod nW)."""
    from paper_2501_06480_b200.shard import shard_images

    sh = shard_images(wl["batch"], 1, rank, world)
    images = sh.images
    out = dict(wl, batch=images,
               layers=[((N // wl["batch"]) * images, h, L, d) for (N, h, L, d) in wl["layers"]])
    return out, images


def measure(args, name, dev, rank, world, dist, steps, with_e2e):
    import torch

    import paper_2501_06480_b200 as fwa
    from paper_2501_06480_b200 import _native as nat

    wl = WORKLOADS[name]
    global_windows = None
    if args.strong:
        global_windows = sum(N for (N, h, L, d) in wl["layers"])
        wl, _ = shard_workload(wl, rank, world)
    work = GpuWorkload(wl, dev, 42 + rank)
    ms_step, launches = timed_graph(torch, nat, work, steps, args.warmup, args.eager,
                                    args.soak_s, world, dist)
    peak, peak_src = load_peaks()
    layers = wl["layers"]
    windows = sum(N for (N, h, L, d) in layers)
    byts = work.bytes_per_step()
    # dominant layer (most bytes) timed alone with a cold L2: the roofline numerator
    dom = max(range(len(layers)), key=lambda i: math.prod(layers[i]))
    N, h, L, d = layers[dom]
    unit_bytes = N * h * L * d * work.eb
    fp = fwa.ops.footprint(N, h, L, d, work.dtype)
    fwd_ms = flushed_launch_ms(torch, work, dom, True, False)
    kern = {"fwd": {"shape": [N, h, L, d], "ms": fwd_ms, "GB/s": 4 * unit_bytes / fwd_ms / 1e6,
                    "kernel": fp["kernel_fwd"]}}
    if wl["bwd"]:
        bwd_ms = flushed_launch_ms(torch, work, dom, False, True)
        kern["bwd"] = {"shape": [N, h, L, d], "ms": bwd_ms, "GB/s": 7 * unit_bytes / bwd_ms / 1e6,
                       "kernel": fp["kernel_bwd"],
                       "note": "includes the deterministic dBias reduce" if wl["extras"] else ""}
    mk = "bwd" if wl["bwd"] else "fwd"
    ncu = load_ncu_traffic().get(f"{name}:{mk}") or {}
    mult = 7 if mk == "bwd" else 4
    streamed = mult * unit_bytes > 2 * L2_BYTES
    if streamed:
        s_ms = streamed_launch_ms(torch, work, dom, mk == "fwd", mk == "bwd")
        kern[mk]["ms_flushed"], kern[mk]["GB/s_flushed"] = kern[mk]["ms"], kern[mk]["GB/s"]
        kern[mk]["ms"], kern[mk]["GB/s"] = s_ms, mult * unit_bytes / s_ms / 1e6
    how = ("CUDA events around 20 back-to-back eager launches of the dominant layer on the "
           "launching stream (its traffic is > 2x L2, so each launch streams from HBM), "
           "average per launch; the L2-flushed single-launch median of 21 is kept as "
           "ms_flushed / GB/s_flushed" if streamed else
           "CUDA events around one eager launch on the launching stream, L2 flushed "
           "(512 MB read) before each launch, median of 21")
    roof = {"bound": "hbm", "achieved": kern[mk]["GB/s"], "peak": peak, "unit": "GB/s",
            "frac": kern[mk]["GB/s"] / peak,
            "traffic": ncu.get("dram_bytes_per_launch"),
            "traffic_source": ncu.get("source", "no committed ncu capture for this launch"),
            "tensor_pipe_pct": ncu.get("tensor_pipe_pct"),
            "issue_active_pct": ncu.get("issue_active_pct"),
            "peak_source": peak_src,
            "kernel": f"{mk} ({kern[mk]['kernel']}) on the dominant layer {kern[mk]['shape']}",
            "algorithmic_bytes_per_launch": mult * unit_bytes,
            "bytes_per_unit": f"{mult}*L*d*{work.eb} = {mult * L * d * work.eb} B",
            "how": how,
            "launches": kern,
            "step_frac": byts / (ms_step / 1e3) / 1e9 / peak}
    total_windows = global_windows if global_windows is not None else windows * world
    out = {"value": total_windows / (ms_step / 1e3), "ms_per_step": ms_step,
           "tflops": work.flops_per_step() * world / (ms_step / 1e3) / 1e12,
           "hbm_frac_step": byts / (ms_step / 1e3) / 1e9 / peak, "roofline": roof,
           "gpu_launches": launches, "algorithmic_bytes_per_step": byts}
    if with_e2e:
        out["e2e"] = e2e(args, work, world, dist, total_windows)
    del work
    torch.cuda.empty_cache()
    return out


def e2e(args, work, world, dist, total_windows):
    """Same metric through the public API on pinned HOST buffers (H2D + kernels + D2H)."""
    import torch

    import paper_2501_06480_b200 as fwa

    wl = work.wl
    host = [tuple(t.cpu().pin_memory() if t is not None else None for t in (q, kk, v, do))
            for (q, kk, v, do, _, _, _, _) in work.bufs]
    r = max(1, wl["layers"][0][3] // 16)

    def run():
        for (qh, kh, vh, doh), (_, _, _, _, bias, mask, _, sc) in zip(host, work.bufs):
            cfg = fwa.TileConfig(r=r, scale=sc)
            _, ctx, _ = fwa.batched_flash_forward(qh, kh, vh, cfg, [fwa.ScratchpadArena(1 << 20)],
                                                  bias=bias, mask=mask)
            if wl["bwd"]:
                fwa.batched_flash_backward(ctx, doh, [fwa.ScratchpadArena(1 << 20)])
    run()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    n = max(1, args.e2e_steps)
    t0 = time.perf_counter()
    for _ in range(n):
        run()
    torch.cuda.synchronize()
    s = (time.perf_counter() - t0) / n
    if world > 1:
        s = max_over_ranks(torch, dist, s, work.dev)
    per = [N * h * L * d * work.eb for (N, h, L, d) in wl["layers"]]
    return {"value": total_windows / s, "unit": "windows/s",
            "h2d_bytes_per_step": (4 if wl["bwd"] else 3) * sum(per),
            "d2h_bytes_per_step": (3 if wl["bwd"] else 1) * sum(per),
            "path": "paper_2501_06480_b200.batched_flash_forward"
                    f"{'/batched_flash_backward' if wl['bwd'] else ''} on pinned host torch "
                    "tensors: chunked H2D / kernel / D2H overlapped on three streams, results "
                    "returned in host memory", "steps": n}


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2501_06480_b200 import _native as nat

    wl = WORKLOADS[args.workload]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; FWA_DIST_BACKEND=gloo lets several ranks share a GPU for a smoke test
    backend = os.environ.get("FWA_DIST_BACKEND", "nccl")
    dev = torch.device("cuda", local % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    nat.load()
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")
    sampler = ClockSampler(int(vis[local]) if len(vis) > local and vis[local].isdigit() else local)
    sampler.start()
    main_res = measure(args, args.workload, dev, rank, world, dist, args.steps, not args.no_e2e)
    # the other BASELINE configs ride on the default run as embedded lines (same method)
    embedded = {}
    if args.workload == "swin_t_fwd" and not args.no_extra:
        for name in EMBEDDED:
            embedded[name] = measure(args, name, dev, rank, world, dist,
                                     max(3, args.steps // 4), False)
    extra = embedded.get("swin_t_fwdbwd")
    blocks = windows_k = None
    if args.workload == "swin_t_fwd" and not args.no_extra and world == 1:
        windows_k = measure_window_copies(dev)
        # SURVEY 8(f)4 / PAPER.md:257-260: the whole (S)W-MSA block, fwd + bwd, on the package's
        # kernels vs the same block in plain PyTorch ops (same weights, bf16, eager)
        from paper_2501_06480_b200.swin import block_speedup

        blocks = [block_speedup(*cfg) for cfg in BLOCKS]
    clocks = sampler.stop()
    validation = None
    if world > 1 and not args.no_validate:
        # 1-GPU vs G-GPU bitwise check of the sharded path over the job's process group
        # (NCCL all_gather of per-window bit hashes; outside every timed region)
        from paper_2501_06480_b200.shard import validate_sharding

        N0, h0, L0, d0 = WORKLOADS[args.workload]["layers"][0]
        validation = validate_sharding(rank, world, dev, (N0, h0, L0, d0),
                                       WORKLOADS[args.workload]["batch"])
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, cores, sample, _, kind = cpu_reference(wl, seconds_target=args.cpu_seconds)
        cpu = {"value": v, "unit": "windows/s", "cores": cores, "kind": kind, "sample": sample}
    if rank == 0:
        line = {
            "metric": f"{METRIC} ({wl['desc']})", "value": main_res["value"], "unit": "windows/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": main_res["ms_per_step"], "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak",
            "vs_baseline": None,
            "dtype": {"float16": "f16", "bfloat16": "bf16"}[wl["dtype"]],
            "data": "synthetic (SplitMix64 U[-1,1), seed 42+rank; random bias table)",
            "config": {"workload": args.workload, "desc": wl["desc"],
                       "images_per_gpu": wl["batch"] if not args.strong else
                       f"{wl['batch'] // world}-{-(-wl['batch'] // world)} (shard of {wl['batch']})",
                       "global_batch": wl["batch"] * (1 if args.strong else world),
                       "layers": [list(x) for x in wl["layers"]],
                       "parallelism": f"dp{world} ("
                                      + (f"strong: {wl['batch']} images split over the ranks"
                                         if args.strong else
                                         f"weak: {wl['batch']} images per GPU")
                                      + ", no collective on the hot path)",
                       "launch": "eager" if args.eager else
                                 "one step captured in a CUDA graph, PDL between kernels",
                       "l2": f"no flush for the step: "
                             f"{main_res['algorithmic_bytes_per_step'] / 1e9:.2f} GB of distinct "
                             "tensors per step (>> 126 MB L2); dominant-launch timing flushes L2 "
                             "(512 MB read) before each launch"},
            "tflops": main_res["tflops"], "hbm_frac_step": main_res["hbm_frac_step"],
            "roofline": main_res["roofline"], "gpu_launches": main_res["gpu_launches"],
            "e2e": main_res.get("e2e"), "cpu_baseline": cpu, "clocks": clocks,
        }
        if validation is not None:
            line["validation"] = validation
        if windows_k is not None:
            line["window_partition"] = windows_k
        if blocks is not None:
            line["swin_block"] = {
                "what": "Swin (S)W-MSA block forward + backward (partition + qkv Linear + window "
                        "attention with rel-pos bias / shift mask + proj Linear + reverse), "
                        "paper_2501_06480_b200.SwinWindowAttention vs the same block in plain "
                        "PyTorch ops with shared weights (TorchSwinWindowAttention), bf16, eager, "
                        "CUDA events, mean of 20 steps",
                "configs": blocks}
        def summary(name, res):
            w = WORKLOADS[name]
            return {"workload": name, "desc": w["desc"], "value": res["value"],
                    "unit": "windows/s", "ms_per_step": res["ms_per_step"],
                    "dtype": {"float16": "f16", "bfloat16": "bf16"}[w["dtype"]],
                    "hbm_frac_step": res["hbm_frac_step"], "tflops": res["tflops"],
                    "roofline": res["roofline"], "gpu_launches": res["gpu_launches"],
                    "layers": [list(x) for x in w["layers"]]}
        if extra is not None:
            line["fwd_bwd"] = summary("swin_t_fwdbwd", extra)
        if embedded:
            line["embedded"] = {n: summary(n, r) for n, r in embedded.items()
                                if n != "swin_t_fwdbwd"}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_reference(args):
    wl = WORKLOADS[args.workload]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if int(os.environ.get("RANK", "0")) != 0:
        return
    v, cores, sample, per_step, kind = cpu_reference(wl, seconds_target=args.cpu_seconds,
                                                     steps=args.steps, warmup=args.warmup)
    print(json.dumps({
        "impl": "reference", "metric": f"{METRIC} ({wl['desc']})", "value": v,
        "unit": "windows/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (SplitMix64 U[-1,1))",
        "config": {"workload": args.workload, "desc": wl["desc"],
                   "note": ("reference CPU path = the unmodified reference package (flashwin "
                            "0.1.0, pip-installed offline from /root/reference/pkg into "
                            "baseline/_ref) through its public batched_flash_forward / "
                            "flash_backward, float64, one process per host core"
                            if kind == "reference" else
                            "reference CPU path = oracle port (oracle/flashwin_oracle.py) of "
                            "flash.py Alg.1/2 in float64 on all host cores (baseline/_ref absent)")},
        "cpu_baseline": {"value": v, "unit": "windows/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": v, "unit": "windows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


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
    ap.add_argument("--no-extra", action="store_true", help="skip the embedded fwd+bwd line")
    ap.add_argument("--eager", action="store_true", help="no CUDA graph for the timed steps")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: split the workload's global batch over the ranks")
    ap.add_argument("--no-validate", action="store_true",
                    help="skip the post-timing 1-GPU vs G-GPU bitwise check (N > 1)")
    ap.add_argument("--soak-s", type=float, default=1.5, help="loaded seconds before timing")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)  # timing rule: at least 3 warm-up steps
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
