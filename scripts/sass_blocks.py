"""Hot SASS blocks of one kernel in an ncu report: python scripts/sass_blocks.py REP KERNEL_REGEX [N]."""
import csv, io, re, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
r = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr, data = r[0], [x for x in r[1:] if len(x) == len(r[0])]
ia, ws = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
num = lambda v: int(v) if v.isdigit() else 0
tot = sum(num(x[ia]) for x in data)
stot = sum(num(x[ws]) for x in data) or 1
print(f"{lines[0][:120]}\ninstructions executed {tot}, stall samples {stot}, sass {len(data)}")
blocks, cur = [], None
for i, x in enumerate(data):
    c = num(x[ia])
    if cur and cur[1] == c:
        cur[2] += 1; cur[3] += num(x[ws]); cur[4].append(x[1].strip())
    else:
        cur = [i, c, 1, num(x[ws]), [x[1].strip()]]; blocks.append(cur)
blocks.sort(key=lambda b: -b[1] * b[2])
for b in blocks[:top]:
    ops = {}
    for s in b[4]:
        t = s.split()
        m = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ops[m] = ops.get(m, 0) + 1
    print(f"idx {b[0]:5d} count {b[1]:9d} len {b[2]:4d} instr {b[1]*b[2]/tot*100:5.1f}% stall {b[3]/stot*100:5.1f}%",
          dict(sorted(ops.items(), key=lambda t: -t[1])[:9]))
