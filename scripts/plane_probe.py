"""Run one 2D direct-tap plan (c4-style line PSF at 256^2 float32, or c2 at 512^2 float64) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1212_2245_b200 as md
which = sys.argv[1] if len(sys.argv) > 1 else "c4"
if which == "c4":
    shape, dtype, n, params = (256, 256), "float32", 512, md.DeconvParams()
    psf = md.Psf.line(17.0, 37.0)
else:
    shape, dtype, n, params = (512, 512), "float64", 64, md.DeconvParams(iterations=10)
    psf = md.Psf.line(21.0, 30.0)
pipe = md.DeblurPipeline(shape, psf, params, dtype=dtype)
tdt = torch.float32 if dtype == "float32" else torch.float64
f = (torch.rand((n,) + shape, device="cuda", dtype=torch.float64) * 200 + 20).to(tdt)
for _ in range(3):
    u = pipe.run_batch(f)
torch.cuda.synchronize()
print(pipe.plan.describe, "ok")
