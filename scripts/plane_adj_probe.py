"""Direct-tap plane path (float64): output hashes over PSF shapes / frame sizes / boundary modes
and the c5 iteration time -- run against two library builds (MD_LIB=...) to check that a stage-
kernel change is bit-identical and to time it (used for the adjacent-column stage-B experiment,
DESIGN.md section 6)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1212_2245_b200 as md

gen = torch.Generator("cuda").manual_seed(9)
cases = [((256, 256), md.Psf.line(15.0, 40.0)), ((256, 256), md.Psf.line(21.0, 30.0)),
         ((256, 256), md.Psf.line(19.0, 100.0)), ((256, 256), md.Psf.line(9.0, 0.0)),
         ((256, 256), md.Psf.general_2d(np.random.default_rng(1).uniform(0, 1, (7, 7)))),
         ((256, 256), md.Psf.general_2d(np.random.default_rng(2).uniform(0, 1, (4, 6)))),
         ((32, 64), md.Psf.line(13.0, 20.0)), ((64, 128), md.Psf.line(21.0, 150.0)),
         ((512, 512), md.Psf.line(21.0, 30.0))]
for shape, psf in cases:
    g = torch.rand((4, *shape), dtype=torch.float64, device="cuda", generator=gen) * 250 + 3
    for sc in (md.Scenario.FOURIER_2D,):
        pipe = md.DeblurPipeline(shape, psf, md.DeconvParams(), sc)
        h = hashlib.sha1(pipe.run_batch(g).cpu().numpy().tobytes()).hexdigest()[:12]
        print(shape, sc.value, h, pipe.plan.describe, flush=True)
# clamped spatial convolver (rrrl_deblur with the spatial mode) on one frame
f = md.Image(torch.rand((96, 160), dtype=torch.float64, generator=torch.Generator().manual_seed(3)).numpy() * 200 + 5)
for psf in (md.Psf.line(11.0, 60.0), md.Psf.line(17.0, 10.0)):
    u = md.rrrl_deblur(f, psf, md.DeconvParams(iterations=3))
    print("spatial", hashlib.sha1(np.asarray(u.values).tobytes()).hexdigest()[:12], flush=True)
# the c5 route at 4096^2 (one plan) and the c5 iteration time at 16384^2
for n in (4096, 16384):
    psf = md.Psf.line(21.0, 30.0)
    g = torch.rand((1, n, n), dtype=torch.float64, device="cuda", generator=gen) * 250 + 3
    pipe = md.DeblurPipeline((n, n), psf, md.DeconvParams(), big_fft=True)
    u = torch.empty_like(g)
    pipe.plan.run(g, out=u)
    h = hashlib.sha1(u.cpu().numpy().tobytes()).hexdigest()[:12]
    ts = sorted(pipe.plan.run_profile(g, out=u)["iter_ms"] for _ in range(3))
    print(f"c5 n={n} {h} iter_ms={ts[1]:.2f}", flush=True)
    del g, u, pipe
    torch.cuda.empty_cache()
