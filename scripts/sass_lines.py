#!/usr/bin/env python
"""Attribute ncu SASS-level stall samples to CUDA source lines.

    python scripts/sass_lines.py REPORT.ncu-rep CUBIN KERNEL_MANGLED [TOP] [COLUMN]

COLUMN (optional): rank lines by that source-page column instead of stall samples, e.g.
"L1 Wavefronts Shared" (shared-memory wavefronts per source line).

The ncu source page (--print-source sass) gives per-instruction samples by runtime address;
nvdisasm --print-line-info of the same cubin maps instruction offsets to file:line. The kernel's
first instruction anchors the offset."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
col = sys.argv[5] if len(sys.argv) > 5 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
# one block per profiled kernel ("Kernel Name" row, then the "Address" header): take the block
# whose name matches the kernel (mangled names contain the demangled base name)
mm = re.match(r"^_ZN\d+md(\d+)", kern)
want = kern[mm.end():mm.end() + int(mm.group(1))] if mm else kern       # e.g. k_fused_lines64
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] or [0]
blk = next((i for i in starts if want in " ".join(rows[i][1:])), starts[0])
hi = next(i for i, r in enumerate(rows) if i >= blk and r and r[0] == "Address")
end = next((i for i in starts if i > hi), len(rows))
rows = rows[:end]
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and not c.endswith("(Not Issued)")]
ri = [h.index(c) for c in reasons]
ci = h.index(col) if col else si


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


sass = [(int(r[0], 16), num(r[ci]), float(r[ie] or 0), r[1].strip(),
         [float(r[i] or 0) for i in ri]) for r in rows[hi + 1:] if len(r) > si]
base = sass[0][0]
dis = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
line_of = {}
cur = None
inside = False
for ln in dis.splitlines():
    if ln.startswith(".text."):
        inside = ln.strip().rstrip(":") == ".text." + kern
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(\S.*)", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: [0.0, 0.0, [0.0] * len(reasons)])
tot = 0.0
overall = [0.0] * len(reasons)
for addr, s, n, _, rs in sass:
    k = line_of.get(addr - base, "?")
    agg[k][0] += s
    agg[k][1] += n
    for j, v in enumerate(rs):
        agg[k][2][j] += v
        overall[j] += v
    tot += s
ts = sum(overall) or 1.0
print("overall:", ", ".join(f"{reasons[j][6:]} {100 * overall[j] / ts:.1f}%"
                            for j in sorted(range(len(reasons)), key=lambda j: -overall[j])[:8]))
print(f"total {sum(a[1] for a in agg.values()) / 1e6:.1f}M warp instructions")
for k, (s, n, rs) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    top3 = sorted(range(len(reasons)), key=lambda j: -rs[j])[:3]
    why = ", ".join(f"{reasons[j][6:]} {100 * rs[j] / max(s, 1):.0f}%" for j in top3)
    extra = f"  {s / 1e6:9.2f}M {col}" if col else ""
    print(f"{100 * s / tot:5.1f}%  {n / 1e6:8.2f}M inst  {k:32s} [{why}]{extra}")
