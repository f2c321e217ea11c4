"""GPU `check` and `traffic` commands.

The reference CLI's correctness / traffic / occupancy suite (pkg/src/flashwin/cli.py:62-145,
harness.py:163-239 `run_check_suite`, :409-466 `run_traffic`) re-run through this
package's drop-in API on the sm_100a kernels:

    python -m paper_2501_06480_b200.check check   [--L 1 2 8 49 64] [--C 16 32 64] [--r 1 2 4 auto]
    python -m paper_2501_06480_b200.check traffic [--L 49] [--C 32] [--r auto] [--dtype f16]

`check` prints the reference's fixed-width table (case, max_err, traffic, sram, status):
window round trips (bitwise, on the GPU), forward / backward per (L, C, r) against a
float64 torch restatement of naive attention (reference.py:69-124; fp32 on the GPU,
so the bar is 1e-5 relative instead of the reference's 1e-10 for f64), the reference's
per-operand traffic counts and closed-form scratchpad peaks, expected CapacityErrors
when the paper footprint exceeds the arena, and r-invariance (bitwise: the kernels do
not depend on r). `sram` additionally requires the kernel's real shared-memory /
TMEM footprint (fwa_footprint) to fit the device.

`traffic` prints the reference's lines (peaks, per-operand loads/stores, closed-form
check) and then what the B200 path actually moves: algorithmic HBM bytes per unit
(fwd 4·L·d·s, bwd 7·L·d·s; the paper's Alg. 2 reads Q and K twice), the kernel that
runs and its SMEM / TMEM, and the ncu-measured DRAM bytes when profiles/ncu_traffic.json
holds a capture of that shape.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from dataclasses import dataclass
from typing import Sequence

import torch

from . import ops
from .api import flash_backward, flash_forward
from .errors import CapacityError, FlashwinError
from .rng import Rng, fill_uniform
from .tiling import (
    DEFAULT_CAPACITY_BYTES,
    ScratchpadArena,
    TileConfig,
    peak_sram_backward,
    peak_sram_forward,
    resolve_r,
)

# harness.py:36-43
ROUNDTRIP_GEOMETRIES = [(4, 4, 1, 2), (6, 6, 2, 3), (8, 8, 4, 2), (14, 14, 3, 7), (224, 224, 3, 7)]
REL_TOL = 1e-5          # fp32 on the GPU vs float64 (north star)
DEFAULT_SEED = 42       # harness.py:35


@dataclass
class SuiteResult:
    """One check case (harness.py:61-69)."""

    case_id: str
    max_err: float
    traffic_ok: bool
    sram_ok: bool
    elapsed_ns: int
    ok: bool


def expected_forward_traffic(L: int, C: int):
    """harness.py:122-123: per-operand element counts of Alg. 1."""
    return {"Q": L * C, "K": L * C, "V": L * C}, {"O": L * C}


def expected_backward_traffic(L: int, C: int):
    """harness.py:126-130: Alg. 2 reads Q and K twice."""
    return ({"Q": 2 * L * C, "K": 2 * L * C, "V": L * C, "dO": L * C},
            {"dQ": L * C, "dK": L * C, "dV": L * C})


def _naive(q, k, v, scale):
    """float64 restatement of reference.py:69-78 (softmax(q k^T scale) v)."""
    return torch.softmax((q @ k.T) * scale, -1) @ v


def _naive_grads(q, k, v, do, scale):
    """float64 restatement of reference.py:94-124 via autograd."""
    qq, kk, vv = (t.clone().requires_grad_(True) for t in (q, k, v))
    _naive(qq, kk, vv, scale).backward(do)
    return qq.grad, kk.grad, vv.grad


def _arr(x):
    """Host result as an ndarray (numpy in -> numpy out; DenseTensor-like -> .array)."""
    return getattr(x, "array", x)


def _rel(a, b: torch.Tensor) -> float:
    a = torch.as_tensor(_arr(a)).to(torch.float64).cpu()
    b = b.to(torch.float64).cpu()
    return float((a - b).abs().max() / max(float(b.abs().max()), 1e-300))


def _device_fits(L: int, C: int, dtype) -> bool:
    fp = ops.footprint(1, 1, L, C, dtype)
    smem_max = torch.cuda.get_device_properties(0).shared_memory_per_block_optin
    return fp["smem_bytes_fwd"] <= smem_max and fp["smem_bytes_bwd"] <= smem_max and \
        fp["tmem_cols_fwd"] <= 512 and fp["tmem_cols_bwd"] <= 512


def _valid_rs(C: int, r_values: Sequence) -> list[int]:
    """harness.py:144-160: resolve, dedupe, drop r that leave an empty chunk."""
    out: list[int] = []
    for value in r_values:
        r = resolve_r(value, C)
        if r in out:
            continue
        try:
            TileConfig(r=r).chunk_width(C)
        except FlashwinError:
            continue
        out.append(r)
    return out


def run_check_suite(seed: int, Ls: Sequence[int], Cs: Sequence[int], r_values: Sequence,
                    capacity_bytes: int = DEFAULT_CAPACITY_BYTES) -> list[SuiteResult]:
    if not Ls or not Cs or not r_values:
        return []
    dev = torch.device("cuda")
    results: list[SuiteResult] = []
    master = Rng(seed)

    for H, W, C, k in ROUNDTRIP_GEOMETRIES:
        t0 = time.perf_counter_ns()
        x = fill_uniform(master.split(), (1, H, W, C), device=dev, dtype=torch.float32)
        y = ops.window_reverse(ops.window_partition(x, k), k, H, W)
        err = float((x - y).abs().max())
        results.append(SuiteResult(f"roundtrip_{H}x{W}x{C}_k{k}", err, True, True,
                                   time.perf_counter_ns() - t0, err == 0.0))

    for L in Ls:
        for C in Cs:
            rng = master.split()
            # host float64 operands (the reference's DenseTensor data); GPU computes in fp32
            q, k, v, do = (fill_uniform(rng, (L, C)).double().cpu().numpy() for _ in range(4))
            tq, tk, tv, tdo = (torch.from_numpy(a) for a in (q, k, v, do))
            fits = _device_fits(L, C, torch.float32)
            outs = []
            for r in _valid_rs(C, r_values):
                cfg = TileConfig(r=r, elem_bytes=4)
                ref_o = _naive(tq, tk, tv, cfg.scale)
                ref_g = _naive_grads(tq, tk, tv, tdo, cfg.scale)
                for kind in ("fwd", "bwd"):
                    t0 = time.perf_counter_ns()
                    need = (peak_sram_forward if kind == "fwd" else peak_sram_backward)(L, C, cfg)
                    if need > capacity_bytes:
                        # expected error: the kernel refuses before any work (flash.py:98-103)
                        try:
                            if kind == "fwd":
                                flash_forward(q, k, v, cfg, ScratchpadArena(capacity_bytes))
                            else:
                                _, ctx, _ = flash_forward(q, k, v, cfg, ScratchpadArena(1 << 40))
                                flash_backward(ctx, do, ScratchpadArena(capacity_bytes))
                            refused = False
                        except CapacityError:
                            refused = True
                        results.append(SuiteResult(f"capacity_{kind}_L{L}_C{C}_r{r}", 0.0, True,
                                                   True, time.perf_counter_ns() - t0, refused))
                        if kind == "fwd":
                            break
                        continue
                    arena = ScratchpadArena(capacity_bytes)
                    if kind == "fwd":
                        o, _, rep = flash_forward(q, k, v, cfg, arena)
                        err = _rel(o, ref_o)
                        exp_l, exp_s = expected_forward_traffic(L, C)
                        outs.append(_arr(o).copy())
                    else:
                        _, ctx, _ = flash_forward(q, k, v, cfg, ScratchpadArena(capacity_bytes))
                        dq, dk, dv, rep = flash_backward(ctx, do, arena)
                        err = max(_rel(a, b) for a, b in zip((dq, dk, dv), ref_g))
                        exp_l, exp_s = expected_backward_traffic(L, C)
                    traffic_ok = rep.loads == exp_l and rep.stores == exp_s
                    sram_ok = rep.peak_sram_bytes == need and fits
                    results.append(SuiteResult(f"{kind}_L{L}_C{C}_r{r}", err, traffic_ok, sram_ok,
                                               time.perf_counter_ns() - t0,
                                               err <= REL_TOL and traffic_ok and sram_ok))
            if len(outs) >= 2:
                t0 = time.perf_counter_ns()
                same = all(bool((o == outs[0]).all()) for o in outs[1:])
                results.append(SuiteResult(f"invariance_L{L}_C{C}", 0.0 if same else 1.0, True,
                                           True, time.perf_counter_ns() - t0, bool(same)))
    return results


def render_suite_table(results: list[SuiteResult]) -> str:
    """harness.py:371-386 format."""
    if not results:
        return "0 cases (empty grid): vacuous pass\n"
    width = max(len(r.case_id) for r in results)
    lines = [f"{'case':<{width}}  {'max_err':>10}  traffic  sram  status"]
    for r in results:
        lines.append(f"{r.case_id:<{width}}  {r.max_err:>10.3e}  "
                     f"{'ok' if r.traffic_ok else 'FAIL':<7}  "
                     f"{'ok' if r.sram_ok else 'FAIL':<4}  {'PASS' if r.ok else 'FAIL'}")
    passed = sum(r.ok for r in results)
    lines.append(f"{passed}/{len(results)} cases passed")
    return "\n".join(lines) + "\n"


_DTYPES = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}


def run_traffic(L: int, C: int, r: int, dtype: str = "f16", units: int = 1,
                seed: int = DEFAULT_SEED, capacity_bytes: int = DEFAULT_CAPACITY_BYTES) -> str:
    """harness.py:409-466 lines, then the B200 path's real bytes and footprint."""
    cfg = TileConfig(r=r, elem_bytes=4)
    rng = Rng(seed)
    q, k, v, do = (fill_uniform(rng, (L, C)).double().cpu().numpy() for _ in range(4))
    pf, pb = peak_sram_forward(L, C, cfg), peak_sram_backward(L, C, cfg)
    # the report needs a run: grow the arena past the paper footprint when it does not fit
    # (the reference would raise CapacityError; the B200 kernels have their own budget)
    cap = max(capacity_bytes, pb)
    _, ctx, fwd = flash_forward(q, k, v, cfg, ScratchpadArena(cap))
    _, _, _, bwd = flash_backward(ctx, do, ScratchpadArena(cap))
    efl, efs = expected_forward_traffic(L, C)
    ebl, ebs = expected_backward_traffic(L, C)
    consistent = (fwd.loads == efl and fwd.stores == efs and bwd.loads == ebl and
                  bwd.stores == ebs and fwd.peak_sram_bytes == pf and bwd.peak_sram_bytes == pb)

    def fmt(c):
        return ", ".join(f"{n}={v}" for n, v in sorted(c.items()))

    dt = _DTYPES[dtype]
    s = torch.tensor([], dtype=dt).element_size()
    fp = ops.footprint(units, 1, L, C, dt)
    lines = [
        f"shape L={L} C={C} r={r} elem_bytes={cfg.elem_bytes}",
        f"forward  peak: {fwd.peak_sram_bytes} B (formula {pf} B, {pf / 1000:.3f} kB)",
        f"backward peak: {bwd.peak_sram_bytes} B (formula {pb} B, {pb / 1000:.3f} kB)",
        f"forward  loads: {fmt(fwd.loads)}",
        f"forward  stores: {fmt(fwd.stores)}",
        f"backward loads: {fmt(bwd.loads)}",
        f"backward stores: {fmt(bwd.stores)}",
        f"instrumented counts match closed form: {'yes' if consistent else 'NO'}",
        *([f"(paper scratchpad {pb} B exceeds the {capacity_bytes} B arena: reported with a "
           f"{cap} B arena)"] if cap > capacity_bytes else []),
        f"B200 {dtype}: forward moves {4 * L * C * s} B/unit (Q, K, V in, O out); backward "
        f"{7 * L * C * s} B/unit (Q, K, V, dO in once, dQ, dK, dV out; the Alg. 2 count "
        f"above reads Q and K twice: {9 * L * C * s} B)",
        f"B200 {dtype}: forward kernel {fp['kernel_fwd']} (smem {fp['smem_bytes_fwd']} B, "
        f"TMEM {fp['tmem_cols_fwd']} cols); backward kernel {fp['kernel_bwd']} "
        f"(smem {fp['smem_bytes_bwd']} B, TMEM {fp['tmem_cols_bwd']} cols)",
    ]
    prof = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "profiles", "ncu_traffic.json")
    try:
        with open(prof) as f:
            caps = json.load(f)
    except (OSError, ValueError):
        caps = {}
    for key, cap in sorted(caps.items()):
        shp = cap.get("shape", [])
        if len(shp) == 4 and shp[2] == L and shp[3] == C:
            n_units = shp[0] * shp[1]
            lines.append(f"ncu {key} {cap.get('dtype')} shape {shp}: "
                         f"{cap['dram_bytes_per_launch'] / n_units:.0f} DRAM B/unit measured vs "
                         f"{cap['algorithmic_bytes_per_launch'] / n_units:.0f} algorithmic")
    return "\n".join(lines) + "\n"


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2501_06480_b200.check")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("check", help="correctness / traffic / occupancy suite on the GPU")
    p.add_argument("--L", type=int, nargs="+", default=[1, 2, 8, 49, 64])
    p.add_argument("--C", type=int, nargs="+", default=[16, 32, 64])
    p.add_argument("--r", nargs="+", default=["1", "2", "4", "auto"])
    p.add_argument("--seed", type=int, default=DEFAULT_SEED)
    p.add_argument("--capacity-bytes", type=int, default=DEFAULT_CAPACITY_BYTES)
    p = sub.add_parser("traffic", help="traffic and footprint for one shape")
    p.add_argument("--L", type=int, default=49)
    p.add_argument("--C", type=int, default=32)
    p.add_argument("--r", default="auto")
    p.add_argument("--dtype", default="f16", choices=sorted(_DTYPES))
    p.add_argument("--seed", type=int, default=DEFAULT_SEED)
    p.add_argument("--capacity-bytes", type=int, default=DEFAULT_CAPACITY_BYTES)
    args = ap.parse_args(argv)
    rs = [v if v == "auto" else int(v) for v in getattr(args, "r", [])] \
        if args.command == "check" else None
    if args.command == "check":
        res = run_check_suite(args.seed, args.L, args.C, rs, args.capacity_bytes)
        sys.stdout.write(render_suite_table(res))
        bad = [r.case_id for r in res if not r.ok]
        if bad:
            print("failing cases: " + ", ".join(bad), file=sys.stderr)
            return 1
        return 0
    r = resolve_r(args.r if args.r == "auto" else int(args.r), args.C)
    sys.stdout.write(run_traffic(args.L, args.C, r, args.dtype, seed=args.seed,
                                 capacity_bytes=args.capacity_bytes))
    return 0


if __name__ == "__main__":
    sys.exit(main())
