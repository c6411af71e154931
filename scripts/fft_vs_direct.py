"""c4 2D class: direct-tap cluster kernel vs the 2D FFT convolver (force_fft2d), float32."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1212_2245_b200 as md
from bench import c4_bank

bank, kinds = c4_bank(md)
n = 1024
f = torch.rand((n, 256, 256), device="cuda") * 200 + 20
u = torch.empty_like(f)
for i in (32, 38, 39, 44):
    for force in (False, True):
        pipe = md.DeblurPipeline((256, 256), bank[i], md.DeconvParams(), dtype="float32", force_fft2d=force)
        pipe.plan.run(f, out=u)
        torch.cuda.synchronize()
        p = pipe.plan.run_profile(f, out=u)
        print(i, "fft" if force else "direct", {k: round(1e3 * v / n, 2) for k, v in p.items() if k.endswith("_ms")}, flush=True)
