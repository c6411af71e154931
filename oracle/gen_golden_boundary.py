"""Generate the drop-in-boundary fixtures tests/golden/bnd_*.npz by running the REFERENCE
package itself (build container only, seconds):

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_boundary.py

* bnd_lut_custom: DivergenceLut.build(delta=1/16, step=1/1000, upper=40, direct_below=0.4)
  (deconv.py:95-112) -- its table and r1 at probe points (deconv.py:114-134);
* bnd_pipe_lut_custom: DeblurPipeline(..., lut=that table).run (deconv.py:611-690), box L=9;
* bnd_rrrl_lut_custom: rrrl_deblur(..., lut=that table) with the general-1D kernel;
* bnd_rrrl_object / bnd_rl_object / bnd_step_object: rrrl_deblur, rl_deblur and
  prepare_state + rrrl_step given a convolver OBJECT (the reference's own _SpatialConvolver,
  deconv.py:295-307, passed in directly -- the duck-typed protocol of deconv.py:456-457, 549-550).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
LUT = dict(delta=1.0 / 16.0, step=1.0 / 1000.0, upper=40.0, direct_below=0.4)


def main() -> None:
    sys.path.insert(0, REF_SRC)
    import motiondeblur as md
    from motiondeblur.core import BlurAxis, Psf
    from motiondeblur.deconv import (DeblurPipeline, DivergenceLut, Scenario, make_convolver, prepare_state,
                                     rl_deblur, rrrl_deblur, rrrl_step)

    def save(name, **arrays):
        path = os.path.join(OUT, name + ".npz")
        np.savez_compressed(path, **arrays)
        print(f"{os.path.getsize(path):>8d}  {name}")

    lut = DivergenceLut.build(**LUT)
    xs = np.concatenate([10 ** np.random.default_rng(9).uniform(-5, 2.5, 3000), [0.0625, 0.4, 0.3999999, 1.0, 40.0,
                                                                                  40.5, 100.0]])
    save("bnd_lut_custom", x=xs, out=lut.r1(xs), table=lut.table, lut=np.array([LUT[k] for k in
                                                                                   ("delta", "step", "upper", "direct_below")]))
    params = md.DeconvParams()
    g = md.make_test_image(64, 64, seed=11)
    box = Psf.uniform_box(BlurAxis.HORIZONTAL, 9)
    f = md.quantize(md.add_gaussian_noise(md.synth_blur(g, box), 5.0, seed=3))
    u = DeblurPipeline(f.shape, box, params, Scenario.BOX_1D, lut=lut).run(f).values
    save("bnd_pipe_lut_custom", f=f.values, out=u)
    g1 = Psf.general_1d(np.array([0.2, 0.5, 1.0, 0.7, 0.3]), BlurAxis.VERTICAL, center=1)
    f1 = md.quantize(md.add_gaussian_noise(md.synth_blur(g, g1), 3.0, seed=4))
    u1 = rrrl_deblur(f1, g1, md.DeconvParams(iterations=4), "fourier", lut=lut).values
    save("bnd_rrrl_lut_custom", f=f1.values, out=u1, psf_weights=g1.weights, psf_center=np.array(g1.center))
    # a convolver OBJECT passed in directly (no transposition, no mode string)
    conv = make_convolver(box, f.shape, "spatial")
    save("bnd_rrrl_object", f=f.values, out=rrrl_deblur(f, box, params, conv).values)
    save("bnd_rl_object", f=f.values, out=rl_deblur(f, box, 6, conv, 0.1).values)
    rng = np.random.default_rng(5)
    us = rng.uniform(1, 255, (64, 64))
    fs = rng.uniform(1, 255, (64, 64))
    st = prepare_state(md.Image(us), md.Image(fs), box, params, conv)
    un = rrrl_step(st, md.Image(fs), box, params, conv).values
    save("bnd_step_object", u=us, f=fs, blurred=st.blurred.values, weight=st.weight.values,
         diffusion=st.diffusion.values, out=un)


if __name__ == "__main__":
    main()
