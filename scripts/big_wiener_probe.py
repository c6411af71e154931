"""Two-level-FFT Wiener (big_fft) vs the single-pass 2D Wiener on the same frame: where do they differ?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1212_2245_b200 as md
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
psf = md.Psf.line(21.0, 30.0)
f = torch.from_numpy(md.synth_blur(md.make_test_image(n, n, seed=7), psf).values.copy()).cuda()
p0 = md.DeblurPipeline((n, n), psf, md.DeconvParams(iterations=0))
p1 = md.DeblurPipeline((n, n), psf, md.DeconvParams(iterations=0), big_fft=True)
a, b = p0.run_batch(f).cpu().numpy(), p1.run_batch(f).cpu().numpy()
d = np.abs(a - b)
print(p0.plan.describe, "|", p1.plan.describe)
print("max", d.max(), "count >1e-9", int((d > 1e-9).sum()), "of", d.size)
if (d > 1e-9).any():
    ys, xs = np.nonzero(d > 1e-9)
    print("rows", np.unique(ys)[:20], "cols", np.unique(xs)[:20])
