"""Summarise ncu raw-page CSV exports (tools/profile_r2.sh) into one JSON per kernel capture:
device time, DRAM bytes, tensor-pipe / issue / MUFU utilisation, L2 throughput."""
import csv
import json
import sys

METRICS = {
    "gpu__time_duration.sum": "time_us",
    "dram__bytes_read.sum": "dram_read_MB",
    "dram__bytes_write.sum": "dram_write_MB",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active": "mufu_xu_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}
SCALE = {"time_us": 1e-3, "dram_read_MB": 1e-6, "dram_write_MB": 1e-6}


def summarise(path):
    rows = list(csv.reader(open(path)))
    i0 = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, units, vals = rows[i0], rows[i0 + 1], rows[i0 + 2]
    out = {"kernel": vals[hdr.index("Kernel Name")][:160]}
    for m, k in METRICS.items():
        if m in hdr:
            v = vals[hdr.index(m)].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                continue
            u = units[hdr.index(m)]
            if k in SCALE:   # normalise to us / MB whatever unit ncu chose
                mult = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "byte": 1e-6, "Kbyte": 1e-3,
                        "Mbyte": 1.0, "Gbyte": 1e3}.get(u, None)
                x = x * mult if mult is not None else x
            out[k] = round(x, 3)
    return out


if __name__ == "__main__":
    res = {p.split("/")[-1].replace(".raw.csv", ""): summarise(p) for p in sys.argv[1:]}
    print(json.dumps(res, indent=1))
