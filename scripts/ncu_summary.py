#!/usr/bin/env python
"""Summarise an ncu --set full report (.ncu-rep) or a launch-list CSV into markdown.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep            # per-kernel key metrics
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv [MIN_CTAS] # time share per kernel
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def rep(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = ["| kernel | " + " | ".join(label for _, label in KEYS) + " |",
           "|---" * (len(KEYS) + 1) + "|"]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0][:60]
        cells = []
        for key, _ in KEYS:
            if key in hdr:
                i = hdr.index(key)
                cells.append(f"{r[i]} {units[i]}".strip())
            else:
                cells.append("n/a")
        out.append(f"| {name} | " + " | ".join(cells) + " |")
    return "\n".join(out)


def launches(path: str, min_ctas: int = 0) -> str:
    """Time share per kernel; min_ctas > 0 keeps only launches with at least that many CTAs
    (drops plan-time and single-frame latency launches from a bench command's list)."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
    agg = collections.OrderedDict()
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[1:]:
        if min_ctas and gi is not None:
            g = [int(x) for x in r[gi].strip("()").split(",")]
            if g[0] * g[1] * g[2] < min_ctas:
                continue
        k = r[ki].split("(")[0]
        agg.setdefault(k, []).append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| {k[:70]} | {len(v)} | {sum(v):.1f} | {sum(v) / len(v):.1f} | {100 * sum(v) / tot:.1f}% |")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(launches(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0))
    else:
        print(rep(sys.argv[1]))
