"""Executed-instruction histogram by SASS opcode for one kernel of an ncu report.
    python scripts/sass_opcodes.py REPORT.ncu-rep KERNEL_SUBSTRING [TOP] [full]"""
import collections, csv, io, re, subprocess, sys
rep, want = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
FULL = len(sys.argv) > 4 and sys.argv[4] == "full"      # keep the opcode modifiers
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
blk = next(i for i in starts if want in " ".join(rows[i][1:]))
hi = next(i for i, r in enumerate(rows) if i >= blk and r and r[0] == "Address")
end = next((i for i in starts if i > hi), len(rows))
h = rows[hi]
ie, src = h.index("Instructions Executed"), h.index("Source")
agg = collections.Counter()
for r in rows[hi + 1:end]:
    if len(r) <= ie:
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+(?:\.[A-Z0-9_.]+)?)" if FULL else r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[src])
    if m:
        agg[m.group(2)] += float(r[ie] or 0)
tot = sum(agg.values())
print(f"total {tot / 1e6:.1f}M warp instructions")
for op, n in agg.most_common(top):
    print(f"{100 * n / tot:5.1f}%  {n / 1e6:9.2f}M  {op}")
