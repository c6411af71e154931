"""2D-FFT convolver path (c3 geometry and a small dense case): output hash and iteration time --
compare across MD_FFT2_DPRE=0/1 or library variants (bit-identity + timing)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1212_2245_b200 as md
yy, xx = np.mgrid[-15:16, -15:16]
w = np.exp(-(yy ** 2 + xx ** 2) / 50.0) * np.random.default_rng(3).uniform(0.2, 1.0, (31, 31))
gen = torch.Generator("cuda").manual_seed(11)
for n, nf in ((1024, 8), (256, 16)):
    pipe = md.DeblurPipeline((n, n), md.Psf.general_2d(w), md.DeconvParams(), dtype="float64")
    f = torch.rand((nf, n, n), device="cuda", dtype=torch.float64, generator=gen) * 200 + 20
    u = torch.empty_like(f)
    pipe.plan.run(f, out=u)
    h = hashlib.sha1(u.cpu().numpy().tobytes()).hexdigest()[:12]
    ts = sorted(pipe.plan.run_profile(f, out=u)["iter_ms"] / nf for _ in range(3))
    print(f"n={n} {h} iter_ms/frame={ts[1]:.3f} {pipe.plan.describe}", flush=True)
