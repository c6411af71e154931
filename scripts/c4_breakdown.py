"""c4 bank: device time per PSF class (all 48 PSFs, the bench's own frames per group).
usage: python scripts/c4_breakdown.py [float32|float64]"""
import os, sys, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import collections
import torch
import paper_1212_2245_b200 as md
from bench import C4

from bench import gpu_synth
dt = sys.argv[1] if len(sys.argv) > 1 else "float32"
work = C4(md, types.SimpleNamespace(dtype=dt, batch=16384), gpu_synth(md))
f_all = work.device_frames(torch.float32 if dt == "float32" else torch.float64)
tot = collections.defaultdict(float)
cnt = collections.Counter()
for b, s, e in work.pipe.groups(work.index):
    plan = work.pipe.pipes[b].plan
    f = f_all[s:e]
    u = torch.empty_like(f)
    plan.run(f, out=u)
    torch.cuda.synchronize()
    p = plan.run_profile(f, out=u)
    n = e - s
    us = 1e3 * (p["init_ms"] + p["iter_ms"] + p["layout_ms"]) / n
    desc = plan.describe
    key = work.kinds[b] + (" fused" if "fused" in desc else " per-it") + (" box" if " box " in desc else "")
    tot[key] += us
    cnt[key] += 1
    print(f"{b:2d} {work.kinds[b]:10s} {us:6.2f} us/frame (init {1e3 * p['init_ms'] / n:5.2f})  {desc[:90]}", flush=True)
allus = sum(tot.values())
for k in sorted(tot):
    print(f"{k:28s} n={cnt[k]:2d} mean {tot[k]/cnt[k]:6.2f} us share {100*tot[k]/allus:5.1f}%")
print(f"bank mean {allus/sum(cnt.values()):.2f} us/frame -> {1e6/(allus/sum(cnt.values())):.0f} frames/s")
