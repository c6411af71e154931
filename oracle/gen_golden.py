"""Generate tests/golden/*.npz by running the REFERENCE package itself (build container only).

Usage (from the repo root, in the build container where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden.py

The reference (``/root/reference/pkg/src/motiondeblur``) is imported in place, read-only.
Each fixture stores the exact input, the PSF description, the parameters, the entry point
that was called and the reference output, so the oracle (``oracle/wr3l_oracle.py``) and
the CUDA path can both be checked against it on a machine without the reference.
Inputs are built with the reference's own synthetic tooling (make_test_image, synth_blur,
quantize, add_gaussian_noise), exactly as SURVEY.md section 8(d) prescribes.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")


def _psf_fields(psf) -> dict:
    d = {
        "psf_kind": np.array(psf.kind.value),
        "psf_weights": np.asarray(psf.weights, dtype=np.float64),
        "psf_center": np.atleast_1d(np.asarray(psf.center, dtype=np.int64)),
        "psf_axis": np.array("" if psf.axis is None else psf.axis.value),
        "psf_length": np.array(np.nan if psf.length is None else psf.length),
    }
    return d


def _params_fields(p) -> dict:
    return {"params": np.array([p.wiener_k, p.alpha, p.iterations, p.eps_data, p.eps_reg,
                                p.floor], dtype=np.float64)}


def _img(a):
    """Store integer-valued images compactly (exact), others as float64."""
    a = np.asarray(a, dtype=np.float64)
    if np.all(a == np.round(a)) and a.min() >= 0 and a.max() <= 255:
        return a.astype(np.uint8)
    return a


def main() -> None:
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, os.path.dirname(HERE))
    import motiondeblur as md
    from motiondeblur.core import BlurAxis, Psf
    from motiondeblur.deconv import DeblurPipeline, Scenario, make_convolver, prepare_state
    from paper_1212_2245_b200.core import Psf as LinePsf   # rasteriser only (host numpy)

    os.makedirs(OUT, exist_ok=True)
    written = []

    def save(name, **arrays):
        path = os.path.join(OUT, name + ".npz")
        np.savez_compressed(path, **arrays)
        written.append((name, os.path.getsize(path)))

    def scene(h, w, seed=7):
        return md.make_test_image(w, h, seed=seed)

    def degrade(g, psf, sigma, seed):
        f = md.synth_blur(g, psf)
        if sigma > 0:
            f = md.quantize(md.add_gaussian_noise(f, sigma, seed=seed))
        return f

    def pipe_case(name, h, w, psf, params, scenario, sigma, seed=5, keep_g=True):
        g = scene(h, w)
        f = degrade(g, psf, sigma, seed)
        u = DeblurPipeline(f.shape, psf, params, scenario).run(f).values
        extra = {"g": _img(g.values)} if keep_g else {}
        save(name, entry=np.array("pipeline"), scenario=np.array(scenario.value),
             f=_img(f.values), out=u, **_psf_fields(psf), **_params_fields(params), **extra)

    dp = md.DeconvParams()
    rng = np.random.default_rng(20261018)

    # --- c1: the headline config at full size (BASELINE.json configs[0]) -------------
    pipe_case("pipe_c1_box_h15_256", 256, 256, Psf.uniform_box(BlurAxis.HORIZONTAL, 15), dp,
              Scenario.BOX_1D, sigma=5.0, seed=5)
    # --- box variants ----------------------------------------------------------------
    pipe_case("pipe_box_v21p5_64x96", 64, 96, Psf.uniform_box(BlurAxis.VERTICAL, 21.5), dp,
              Scenario.BOX_1D, sigma=5.0, seed=6)
    pipe_case("pipe_box_h9_iter0_64x128", 64, 128, Psf.uniform_box(BlurAxis.HORIZONTAL, 9),
              md.DeconvParams(iterations=0), Scenario.BOX_1D, sigma=0.0)
    pipe_case("pipe_box_h15_alpha0_64", 64, 64, Psf.uniform_box(BlurAxis.HORIZONTAL, 15),
              md.DeconvParams(alpha=0.0, iterations=4), Scenario.BOX_1D, sigma=5.0, seed=8)
    pipe_case("pipe_box_h4_128x32", 128, 32, Psf.uniform_box(BlurAxis.HORIZONTAL, 4), dp,
              Scenario.BOX_1D, sigma=5.0, seed=9)
    # --- general 1D (FOURIER_1D) -----------------------------------------------------
    w9 = rng.uniform(0.0, 1.0, 9)
    pipe_case("pipe_f1d_v9_128x64", 128, 64, Psf.general_1d(w9, BlurAxis.VERTICAL, center=3),
              dp, Scenario.FOURIER_1D, sigma=5.0, seed=10)
    w7 = rng.uniform(0.0, 1.0, 7)
    pipe_case("pipe_f1d_h7_64x128", 64, 128, Psf.general_1d(w7, BlurAxis.HORIZONTAL), dp,
              Scenario.FOURIER_1D, sigma=5.0, seed=11)
    pipe_case("pipe_f1d_box_v27_256", 256, 256, Psf.general_1d(md.materialize_box_kernel(27),
              BlurAxis.VERTICAL), dp, Scenario.FOURIER_1D, sigma=0.0)
    # --- general 2D (FOURIER_2D) -----------------------------------------------------
    line = LinePsf.line(21.0, 30.0)
    pipe_case("pipe_f2d_line21_30_128", 128, 128, Psf.general_2d(line.weights, line.center),
              md.DeconvParams(iterations=10), Scenario.FOURIER_2D, sigma=0.0)
    yy, xx = np.mgrid[-15:16, -15:16]
    g31 = np.exp(-(yy ** 2 + xx ** 2) / 50.0) * np.random.default_rng(3).uniform(0.2, 1.0, (31, 31))
    pipe_case("pipe_f2d_gauss31_128", 128, 128, Psf.general_2d(g31), dp, Scenario.FOURIER_2D,
              sigma=0.0)
    pipe_case("pipe_f2d_3x5_64x128", 64, 128, Psf.general_2d(np.ones((3, 5)), center=(0, 3)),
              md.DeconvParams(iterations=3), Scenario.FOURIER_2D, sigma=5.0, seed=12)
    pipe_case("pipe_f2d_boxv9_64", 64, 64, Psf.uniform_box(BlurAxis.VERTICAL, 9), dp,
              Scenario.FOURIER_2D, sigma=5.0, seed=13)

    # --- rrrl_deblur / rl_deblur (deconv.py:524-559) ---------------------------------
    def deblur_case(name, entry, h, w, psf, params, mode, sigma, seed):
        g = scene(h, w)
        f = degrade(g, psf, sigma, seed)
        if entry == "rrrl":
            u = md.rrrl_deblur(f, psf, params, mode).values
        else:
            u = md.rl_deblur(f, psf, params.iterations, mode).values
        save(name, entry=np.array(entry), mode=np.array("" if mode is None else mode),
             f=_img(f.values), out=u, **_psf_fields(psf), **_params_fields(params))

    deblur_case("rrrl_box_v11_64", "rrrl", 64, 64, Psf.uniform_box(BlurAxis.VERTICAL, 11), dp,
                None, 5.0, 21)
    deblur_case("rrrl_box_h6p5_48x64", "rrrl", 48, 64, Psf.uniform_box(BlurAxis.HORIZONTAL, 6.5),
                dp, None, 5.0, 22)
    deblur_case("rrrl_spatial_2d_5x3_40x56", "rrrl", 40, 56,
                Psf.general_2d(rng.uniform(0, 1, (5, 3)), center=(1, 2)), dp, None, 5.0, 23)
    deblur_case("rrrl_spatial_1dh_48", "rrrl", 48, 48,
                Psf.general_1d(rng.uniform(0, 1, 6), BlurAxis.HORIZONTAL, center=4), dp, None,
                5.0, 24)
    deblur_case("rrrl_fourier_1dv_64x32", "rrrl", 64, 32,
                Psf.general_1d(rng.uniform(0, 1, 5), BlurAxis.VERTICAL), dp, "fourier", 5.0, 25)
    deblur_case("rrrl_fourier2d_64", "rrrl", 64, 64, Psf.general_2d(rng.uniform(0, 1, (4, 4))),
                md.DeconvParams(iterations=3), "fourier", 0.0, 26)
    deblur_case("rl_box_v7_64", "rl", 64, 64, Psf.uniform_box(BlurAxis.VERTICAL, 7),
                md.DeconvParams(iterations=8), None, 5.0, 27)
    deblur_case("rl_spatial_2d_32", "rl", 32, 32, Psf.general_2d(rng.uniform(0, 1, (3, 3))),
                md.DeconvParams(iterations=6), None, 5.0, 28)

    # --- component fixtures ------------------------------------------------------------
    a = rng.uniform(0, 255, (64, 128))
    hb = Psf.uniform_box(BlurAxis.HORIZONTAL, 9)
    save("comp_wiener1d_h9", entry=np.array("wiener_1d"), f=a, k=np.array(0.01),
         out=md.wiener_1d(md.Image(a), hb, 0.01).values, **_psf_fields(hb))
    g1 = Psf.general_1d(rng.uniform(0, 1, 7), BlurAxis.VERTICAL, center=2)
    a2 = rng.uniform(0, 255, (128, 48))
    save("comp_wiener1d_v7", entry=np.array("wiener_1d"), f=a2, k=np.array(0.006),
         out=md.wiener_1d(md.Image(a2), g1, 0.006).values, **_psf_fields(g1))
    p2 = Psf.general_2d(rng.uniform(0, 1, (5, 5)))
    a3 = rng.uniform(0, 255, (64, 64))
    save("comp_wiener2d_5x5", entry=np.array("wiener_2d"), f=a3, k=np.array(0.01),
         out=md.wiener_2d(md.Image(a3), p2, 0.01).values, **_psf_fields(p2))
    for ax in (BlurAxis.VERTICAL, BlurAxis.HORIZONTAL):
        for L in (5, 21.5, 27):
            pb = Psf.uniform_box(ax, L)
            a4 = rng.uniform(0, 255, (80, 72))
            tag = f"{ax.value}{str(L).replace('.', 'p')}"
            save(f"comp_box_{tag}", entry=np.array("box_convolve"), f=a4,
                 out=md.box_convolve(md.Image(a4), pb).values, **_psf_fields(pb))
    ps = Psf.general_2d(rng.uniform(0, 1, (3, 4)), center=(1, 2))
    a5 = rng.uniform(0, 255, (16, 12))
    save("comp_spatial_2d_3x4", entry=np.array("spatial_convolve"), f=a5,
         out=md.spatial_convolve(md.Image(a5), ps).values, **_psf_fields(ps))
    ph = Psf.general_1d(rng.uniform(0, 1, 6), BlurAxis.HORIZONTAL, center=4)
    a6 = rng.uniform(0, 255, (8, 24))
    save("comp_spatial_1dh_6", entry=np.array("spatial_convolve"), f=a6,
         out=md.spatial_convolve(md.Image(a6), ph).values, **_psf_fields(ph))
    pf = Psf.general_2d(rng.uniform(0, 1, (5, 3)), center=(3, 1))
    a7 = rng.uniform(0, 255, (32, 64))
    save("comp_fourier_2d_5x3", entry=np.array("fourier_convolve"), f=a7,
         out=md.fourier_convolve(md.Image(a7), pf).values, **_psf_fields(pf))
    pv = Psf.general_1d(rng.uniform(0, 1, 9), BlurAxis.VERTICAL, center=6)
    a8 = rng.uniform(0, 255, (64, 20))
    save("comp_fourier_1dv_9", entry=np.array("fourier_convolve"), f=a8,
         out=md.fourier_convolve(md.Image(a8), pv).values, **_psf_fields(pv))
    fw = rng.uniform(0.0, 255.0, (32, 32))
    fw[0, :8] = [0.0, 0.05, 0.09, 0.1, 0.5, 3.0, 255.0, 0.0]
    bw = rng.uniform(0.02, 400.0, (32, 32))
    bw[0, :8] = [3.0, 0.02, 1e-6, 7.0, 1e-3, 250.0, 1e-5, 900.0]
    save("comp_robust_weight", entry=np.array("robust_weight"), f=fw, b=bw,
         out=md.robust_weight(md.Image(fw), md.Image(bw), eps_data=1.0, floor=0.1).values)
    du = rng.uniform(0, 255, (24, 20))
    save("comp_diffusion", entry=np.array("diffusion_term"), f=du, eps=np.array(0.01),
         out=md.diffusion_term(md.Image(du), 0.01).values,
         energy=np.array(md.diffusion_energy(md.Image(du), 0.01)))
    # one prepare_state + rrrl_step with the box convolver (deconv.py:477-509)
    pbx = Psf.uniform_box(BlurAxis.VERTICAL, 9)
    us = rng.uniform(1, 255, (64, 64))
    fs = rng.uniform(1, 255, (64, 64))
    conv = make_convolver(pbx, us.shape, "box")
    st = prepare_state(md.Image(us), md.Image(fs), pbx, dp, conv)
    un = md.rrrl_step(st, md.Image(fs), pbx, dp, conv).values
    save("comp_rrrl_step_box_v9", entry=np.array("rrrl_step"), u=us, f=fs, blurred=st.blurred.values,
         weight=st.weight.values, diffusion=st.diffusion.values, out=un, **_psf_fields(pbx),
         **_params_fields(dp))
    # divergence table probe points (deconv.py:114-134)
    xs = np.concatenate([10 ** np.random.default_rng(4).uniform(-6, 3, 4000),
                         [0.03125, 0.5, 0.4999999, 1.0, 64.99, 65.0, 65.0001, 200.0]])
    save("comp_lut_r1", entry=np.array("lut_r1"), x=xs, out=md.default_divergence_lut().r1(xs))

    total = 0
    for name, size in written:
        total += size
        print(f"{size:>9d}  {name}")
    print(f"{total:>9d}  total bytes in {OUT}")


if __name__ == "__main__":
    main()
