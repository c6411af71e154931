"""Timing probe of the single-image large-frame path (c5 geometry) on one GPU."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1212_2245_b200 as md

for n in [int(a) for a in sys.argv[1:]] or [4096, 16384]:
    psf = md.Psf.line(21.0, 30.0)
    f = torch.rand(n, n, dtype=torch.float64, device="cuda") * 200 + 20
    pipe = md.DeblurPipeline((n, n), psf, md.DeconvParams())
    print(pipe.plan.describe, flush=True)
    u = pipe.run_batch(f)
    torch.cuda.synchronize()
    for _ in range(2):
        p = pipe.plan.run_profile(f, out=u)
    print(n, p, flush=True)
