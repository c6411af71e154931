import hashlib, os, sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1212_2245_b200 as md
g = torch.rand((16, 256, 256), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(9)) * 250 + 3
for psf in [md.Psf.line(15.0, 40.0), md.Psf.line(21.0, 30.0)]:
    pipe = md.DeblurPipeline((256, 256), psf, md.DeconvParams(), md.Scenario.FOURIER_2D)
    print(hashlib.sha1(pipe.run_batch(g).cpu().numpy().tobytes()).hexdigest()[:12], pipe.plan.describe)
