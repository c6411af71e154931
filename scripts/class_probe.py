"""Per-class timing probe: c4 bank classes (float32) and the c2 / c3 single-frame configs (float64)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1212_2245_b200 as md
from bench import c4_bank

def probe(name, shape, psf, params, dtype, nframes, **kw):
    pipe = md.DeblurPipeline(shape, psf, params, dtype=dtype, **kw)
    tdt = torch.float32 if dtype == "float32" else torch.float64
    f = (torch.rand((nframes,) + shape, device="cuda", dtype=torch.float64) * 200 + 20).to(tdt)
    u = torch.empty_like(f)
    for _ in range(2):
        pipe.plan.run(f, out=u)
    torch.cuda.synchronize()
    acc = {"init_ms": 0, "iter_ms": 0, "layout_ms": 0}
    reps = 5
    for _ in range(reps):
        p = pipe.plan.run_profile(f, out=u)
        for k in acc:
            acc[k] += p[k] / reps
    per = {k: 1e3 * v / nframes for k, v in acc.items()}
    print(f"{name:40s} {pipe.plan.describe[:70]:70s} us/frame init {per['init_ms']:.2f} iter {per['iter_ms']:.2f} "
          f"layout {per['layout_ms']:.2f} -> {1e3 / sum(per.values()):.0f} frames/s", flush=True)

bank, kinds = c4_bank(md)
params = md.DeconvParams()
for i in (0, 1, 3, 16, 17, 32, 33, 44):
    probe(f"c4[{i}] {kinds[i]}", (256, 256), bank[i], params, "float32", 2048)
probe("c2 512 line f64 10it", (512, 512), md.Psf.line(21.0, 30.0), md.DeconvParams(iterations=10), "float64", 64)
yy, xx = np.mgrid[-15:16, -15:16]
w = np.exp(-(yy ** 2 + xx ** 2) / 50.0) * np.random.default_rng(3).uniform(0.2, 1.0, (31, 31))
probe("c3 1024 31x31 f64", (1024, 1024), md.Psf.general_2d(w), params, "float64", 8)
