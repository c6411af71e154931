"""Fused 2D-plane kernel probe: one c4 line-PSF group, timing + max active clusters."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1212_2245_b200 as md
from bench import c4_bank

bank, kinds = c4_bank(md)
n = int(os.environ.get("FP_FRAMES", "1024"))
for i in (32, 33, 44):
    pipe = md.DeblurPipeline((256, 256), bank[i], md.DeconvParams(), dtype="float32")
    f = (torch.rand((n, 256, 256), device="cuda") * 200 + 20)
    u = torch.empty_like(f)
    for _ in range(2):
        pipe.plan.run(f, out=u)
    torch.cuda.synchronize()
    p = pipe.plan.run_profile(f, out=u)
    print(i, pipe.plan.describe, {k: round(1e3 * v / n, 2) for k, v in p.items() if k.endswith("_ms")}, flush=True)
