"""One c4 2D-class PSF group (256^2 float64 frames, line PSF): device time of the Wiener init and
the iterations, for ncu launch lists.  python scripts/c4_2d_probe.py [frames]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1212_2245_b200 as md
nf = int(sys.argv[1]) if len(sys.argv) > 1 else 341
psf = md.Psf.line(15.0, 40.0)
g = torch.rand((nf, 256, 256), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3)) * 255
pipe = md.DeblurPipeline((256, 256), psf, md.DeconvParams(), md.Scenario.FOURIER_2D)
print(pipe.plan.describe)
out = pipe.run_batch(g)
torch.cuda.synchronize()
for it in (0, 5):
    p = md.DeblurPipeline((256, 256), psf, md.DeconvParams(iterations=it), md.Scenario.FOURIER_2D)
    p.run_batch(g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        p.run_batch(g)
    e1.record()
    e1.synchronize()
    print(f"iterations={it}: {e0.elapsed_time(e1) / 3 / nf * 1000:.2f} us/frame")
