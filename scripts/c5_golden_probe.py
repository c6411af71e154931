"""Errors of the 4096^2 c5 run against the reference fixture (tests/golden/big_c5_4096.npz)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1212_2245_b200 as md
d = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/big_c5_4096.npz"))
psf = md.Psf.general_2d(d["psf_weights"], center=tuple(int(c) for c in d["psf_center"]))
g = md.make_test_image(4096, 4096, seed=7).values
f = torch.from_numpy(md.synth_blur(md.Image(g), psf).values.copy()).cuda()
for big in (True, False):
    u = md.DeblurPipeline((4096, 4096), psf, md.DeconvParams(), md.Scenario.FOURIER_2D, big_fft=big).run_batch(f).cpu().numpy()
    er = np.abs(u[d["rows"]] - d["row_values"])
    ep = np.abs(u[d["py"], d["px"]] - d["pix_values"])
    i = np.unravel_index(er.argmax(), er.shape)
    print("big" if big else "small", "rows max", er.max(), "at", d["rows"][i[0]], i[1], "pix max", ep.max(), "rows>1e-6", int((er > 1e-6).sum()))
