"""c3 geometry probe (1024^2, dense 31x31 PSF, float64): a few frames through the 2D FFT convolver."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1212_2245_b200 as md

yy, xx = np.mgrid[-15:16, -15:16]
w = np.exp(-(yy ** 2 + xx ** 2) / 50.0) * np.random.default_rng(3).uniform(0.2, 1.0, (31, 31))
pipe = md.DeblurPipeline((1024, 1024), md.Psf.general_2d(w), md.DeconvParams(), dtype="float64")
f = torch.rand((int(os.environ.get("C3_FRAMES", "4")), 1024, 1024), device="cuda", dtype=torch.float64) * 200 + 20
u = torch.empty_like(f)
for _ in range(2):
    pipe.plan.run(f, out=u)
torch.cuda.synchronize()
p = pipe.plan.run_profile(f, out=u)
print(pipe.plan.describe, {k: round(v / f.shape[0], 3) for k, v in p.items() if k.endswith("_ms")}, flush=True)
