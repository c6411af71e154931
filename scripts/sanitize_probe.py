"""Small runs of the cluster-resident kernels for compute-sanitizer (memcheck / synccheck /
racecheck): k_fused_lines64 (float64, box and dense taps), k_fused_lines (float32 box),
k_fused_plane (float32 2D line PSF). A few frames each, then a parity check so a run that
the sanitizer perturbs still has to be right."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1212_2245_b200 as md
from oracle import wr3l_oracle as O

frames = int(os.environ.get("SAN_FRAMES", "3"))
cases = [
    ("f64 box L=15", md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15), "float64", md.Scenario.BOX_1D),
    ("f64 box L=9.5 vertical", md.Psf.uniform_box(md.BlurAxis.VERTICAL, 9.5), "float64", md.Scenario.BOX_1D),
    ("f64 taps periodic", md.Psf.general_1d(np.linspace(1, 0.2, 7), md.BlurAxis.HORIZONTAL, center=2), "float64",
     md.Scenario.FOURIER_1D),
    ("f32 box L=15", md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15), "float32", md.Scenario.BOX_1D),
    ("f32 2D line", md.Psf.line(9.0, 30.0), "float32", md.Scenario.FOURIER_2D),
]
for name, psf, dt, scen in cases:
    pipe = md.DeblurPipeline((256, 256), psf, md.DeconvParams(), scen, dtype=dt)
    g = md.make_test_image(256, 256)
    f = md.quantize(md.add_gaussian_noise(md.synth_blur(g, psf), 5.0, seed=1))
    x = torch.from_numpy(np.stack([f.values] * frames)).cuda().to(torch.float64 if dt == "float64" else torch.float32)
    out = pipe.plan.run(x).cpu().numpy().astype(np.float64)
    torch.cuda.synchronize()
    if psf.kind is md.PsfKind.UNIFORM_BOX_1D:
        op = O.make_psf("box", axis="h" if psf.axis is md.BlurAxis.HORIZONTAL else "v", length=psf.length)
    elif psf.kind is md.PsfKind.GENERAL_1D:
        op = O.OPsf("1d", np.asarray(psf.weights), int(psf.center), "h")
    else:
        op = O.OPsf("2d", np.asarray(psf.weights), tuple(psf.center))
    ref = O.pipeline(f.values, op, O.OParams(), scen.value)
    err = float(np.abs(out - ref[None]).max())
    print(f"{name}: plan [{pipe.plan.describe}] max|d| vs oracle {err:.3g}", flush=True)
    assert err <= 1e-4 * 255
print("sanitize probe ok")
