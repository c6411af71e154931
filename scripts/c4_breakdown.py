"""c4 bank: device time per PSF class (all 48 PSFs, bench-sized groups), float32."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import collections
import torch
import paper_1212_2245_b200 as md
from bench import c4_bank

bank, kinds = c4_bank(md)
n = int(os.environ.get("C4_GROUP", "341"))
f = torch.rand((n, 256, 256), device="cuda") * 200 + 20
u = torch.empty_like(f)
tot = collections.defaultdict(float)
cnt = collections.Counter()
for i, psf in enumerate(bank):
    pipe = md.DeblurPipeline((256, 256), psf, md.DeconvParams(), dtype="float32")
    pipe.plan.run(f, out=u)
    torch.cuda.synchronize()
    p = pipe.plan.run_profile(f, out=u)
    us = 1e3 * (p["init_ms"] + p["iter_ms"] + p["layout_ms"]) / n
    desc = pipe.plan.describe
    key = kinds[i] + (" fused" if "fused" in desc else " per-it") + (" box" if " box " in desc else "")
    tot[key] += us
    cnt[key] += 1
    print(f"{i:2d} {kinds[i]:10s} {us:6.2f} us/frame  {desc[:90]}", flush=True)
allus = sum(tot.values())
for k in sorted(tot):
    print(f"{k:28s} n={cnt[k]:2d} mean {tot[k]/cnt[k]:6.2f} us share {100*tot[k]/allus:5.1f}%")
print(f"bank mean {allus/len(bank):.2f} us/frame -> {1e6/(allus/len(bank)):.0f} frames/s")
