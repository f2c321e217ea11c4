"""Generate golden vectors by running the REAL reference package ``flashwin``.

Run in the build container (the reference is mounted read-only there; it does
not exist on the GPU box, so the outputs are committed as fixtures):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (small, committed):
  tests/golden/reference_golden.npz   per-case arrays (inputs are regenerated
                                       from seeds by the oracle's SplitMix64)
  tests/golden/reference_golden.json  scalar KATs and cfg1 checksums

Every value here comes from calling flashwin itself:
  Rng/fill_uniform (tensor.py:74-138), naive_forward/backward (reference.py:69-124),
  flash_forward/flash_backward (flash.py:141-266), peak_sram_* (flash.py:84-95),
  window_partition (windowing.py:44-54).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)

import flashwin as fw  # noqa: E402  (the reference)

HERE = os.path.dirname(os.path.abspath(__file__))


def rand(rng, shape):
    return fw.fill_uniform(rng, shape, -1.0, 1.0)


def main() -> None:
    arrays: dict[str, np.ndarray] = {}
    scalars: dict[str, object] = {}

    # --- SplitMix64 KATs (tensor.py) -------------------------------------
    r = fw.Rng(42)
    scalars["rng42_u64"] = [hex(r.next_u64()) for _ in range(3)]
    scalars["fill42_4"] = rand(fw.Rng(42), (4,)).array.tolist()
    r = fw.Rng(7)
    child = r.split()
    scalars["rng7_split_child_u64"] = hex(child.next_u64())
    scalars["rng7_after_split_u64"] = hex(r.next_u64())
    arrays["fill_seed123_37x5"] = fw.fill_uniform(fw.Rng(123), (37, 5), -2.0, 3.0).array

    # --- Single-unit oracle grid (test_acceptance.py:33-81 seeds) -----------
    grid = []
    for L in (1, 2, 8, 49, 64):
        for C in (4, 10, 16, 32, 64):
            seed = 9000 + 100 * L + C
            rng = fw.Rng(seed)
            q, k, v, do = (rand(rng, (L, C)) for _ in range(4))
            for scale in (1.0, 1.0 / np.sqrt(C)):
                o, cache = fw.naive_forward(q, k, v, fw.AttnParams(scale=float(scale)))
                dq, dk, dv = fw.naive_backward(q, k, v, cache, do, fw.AttnParams(scale=float(scale)))
                tag = f"L{L}_C{C}_s{'1' if scale == 1.0 else 'r'}"
                arrays[f"naive_o_{tag}"] = o.array
                arrays[f"naive_dq_{tag}"] = dq.array
                arrays[f"naive_dk_{tag}"] = dk.array
                arrays[f"naive_dv_{tag}"] = dv.array
                # tiled Alg. 1/2 at r = auto (harness.py:115-119)
                rr = max(1, C // 16)
                cfg = fw.TileConfig(r=rr, scale=float(scale))
                arena = fw.ScratchpadArena(1 << 22)
                fo, ctx, frep = fw.flash_forward(q, k, v, cfg, arena)
                fdq, fdk, fdv, brep = fw.flash_backward(ctx, do, fw.ScratchpadArena(1 << 22))
                arrays[f"flash_o_{tag}"] = fo.array
                arrays[f"flash_dq_{tag}"] = fdq.array
                arrays[f"flash_dk_{tag}"] = fdk.array
                arrays[f"flash_dv_{tag}"] = fdv.array
                grid.append(
                    {
                        "L": L, "C": C, "seed": seed, "scale": float(scale), "r": rr, "tag": tag,
                        "fwd_loads": frep.loads, "fwd_stores": frep.stores,
                        "fwd_peak": frep.peak_sram_bytes,
                        "bwd_loads": brep.loads, "bwd_stores": brep.stores,
                        "bwd_peak": brep.peak_sram_bytes,
                    }
                )
    scalars["grid"] = grid

    # --- Peak KATs (test_flash.py:64-84) ----------------------------------
    peaks = []
    for L, C, rr, eb in [(64, 64, 4, 4), (49, 32, 2, 4), (8, 4, 2, 8), (144, 32, 2, 4),
                         (256, 32, 2, 4), (1024, 32, 2, 4), (16, 32, 32, 4), (32, 48, 1, 4)]:
        cfg = fw.TileConfig(r=rr, elem_bytes=eb)
        peaks.append({"L": L, "C": C, "r": rr, "elem_bytes": eb,
                      "fwd": fw.peak_sram_forward(L, C, cfg),
                      "bwd": fw.peak_sram_backward(L, C, cfg)})
    scalars["peaks"] = peaks

    # --- cfg1 (BASELINE configs[0]): (64,3,49,32), q,k,v,dO = 4 draws of Rng(42)
    shape = (64, 3, 49, 32)
    rng = fw.Rng(42)
    q, k, v, do = (rand(rng, shape) for _ in range(4))
    for scale, tag in ((1.0, "s1"), (32 ** -0.5, "sr")):
        params = fw.AttnParams(scale=scale)
        osum = np.zeros(shape)
        dqs, dks, dvs = np.zeros(shape), np.zeros(shape), np.zeros(shape)
        for b in range(shape[0]):
            for h in range(shape[1]):
                sl = lambda t: fw.DenseTensor(shape[2:], t.array[b, h])  # noqa: E731
                o, cache = fw.naive_forward(sl(q), sl(k), sl(v), params)
                dq, dk, dv = fw.naive_backward(sl(q), sl(k), sl(v), cache, sl(do), params)
                osum[b, h], dqs[b, h], dks[b, h], dvs[b, h] = o.array, dq.array, dk.array, dv.array
        scalars[f"cfg1_{tag}"] = {
            "sum_o": float(osum.sum()), "sum_abs_o": float(np.abs(osum).sum()),
            "o_0_0_0_first3": osum[0, 0, 0, :3].tolist(),
            "sum_dq": float(dqs.sum()), "sum_dk": float(dks.sum()), "sum_dv": float(dvs.sum()),
            "sum_abs_dq": float(np.abs(dqs).sum()), "sum_abs_dk": float(np.abs(dks).sum()),
            "sum_abs_dv": float(np.abs(dvs).sum()),
        }
        # two full units as arrays for elementwise pinning
        arrays[f"cfg1_{tag}_o_b0"] = osum[0]
        arrays[f"cfg1_{tag}_o_b63"] = osum[63]
        arrays[f"cfg1_{tag}_dq_b5"] = dqs[5]
        arrays[f"cfg1_{tag}_dk_b5"] = dks[5]
        arrays[f"cfg1_{tag}_dv_b5"] = dvs[5]

    # batched_flash_forward merged report (test_flash.py:271-281)
    rng = fw.Rng(70)
    bq, bk, bv = (rand(rng, (4, 4, 64, 64)) for _ in range(3))
    bo, _, brep = fw.batched_flash_forward(bq, bk, bv, fw.TileConfig(r=4), [fw.ScratchpadArena()])
    scalars["batched70"] = {"loads": brep.loads, "stores": brep.stores,
                            "peak": brep.peak_sram_bytes, "sum_o": float(bo.array.sum())}

    # --- windowing (windowing.py:44-70) -------------------------------------
    vals = np.arange(16.0).reshape(4, 4, 1)
    y = fw.window_partition(fw.DenseTensor((4, 4, 1), vals), fw.WindowConfig(4, 4, 1, 2))
    arrays["win_4x4_k2"] = y.array
    x = rand(fw.Rng(7), (10, 15, 4))
    arrays["win_10x15x4_k5"] = fw.window_partition(x, fw.WindowConfig(10, 15, 4, 5)).array
    x = rand(fw.Rng(0), (56, 56, 8))
    arrays["win_56x56x8_k7"] = fw.window_partition(x, fw.WindowConfig(56, 56, 8, 7)).array

    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **arrays)
    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(scalars, f, indent=1, sort_keys=True)
    print(f"wrote {len(arrays)} arrays, {len(scalars)} scalar groups")


if __name__ == "__main__":
    main()
