"""Pin the CPU oracle (oracle/wr3l_oracle.py) against fixtures produced by the reference.

Every fixture in tests/golden was written by oracle/gen_golden.py running the reference
package itself; the oracle must reproduce each within float64 rounding.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_names, load_golden, oracle_params, oracle_psf
from oracle import wr3l_oracle as O

PIPE = golden_names("pipe_")
DEBLUR = golden_names("rrrl_") + golden_names("rl_")


@pytest.mark.parametrize("name", PIPE)
def test_pipeline_matches_reference(name):
    d = load_golden(name)
    out = O.pipeline(d["f"], oracle_psf(d), oracle_params(d), str(d["scenario"]))
    np.testing.assert_allclose(out, d["out"], rtol=0, atol=1e-8)


@pytest.mark.parametrize("name", DEBLUR)
def test_deblur_entry_matches_reference(name):
    d = load_golden(name)
    psf, params = oracle_psf(d), oracle_params(d)
    mode = str(d["mode"]) or None
    if str(d["entry"]) == "rrrl":
        out = O.rrrl_deblur(d["f"], psf, params, mode)
    else:
        out = O.rl_deblur(d["f"], psf, params.iterations, mode, params.floor)
    np.testing.assert_allclose(out, d["out"], rtol=0, atol=1e-8)


def test_c1_psnr_and_range():
    d = load_golden("pipe_c1_box_h15_256")
    out = O.pipeline(d["f"], oracle_psf(d), oracle_params(d), "box")
    assert abs(O.psnr(out, d["g"]) - O.psnr(d["out"], d["g"])) < 1e-9
    assert out.min() > 0.0


@pytest.mark.parametrize("name", golden_names("comp_"))
def test_components_match_reference(name):
    d = load_golden(name)
    entry = str(d["entry"])
    if entry == "lut_r1":
        np.testing.assert_allclose(O.r1(d["x"]), d["out"], rtol=0, atol=1e-12)
        return
    if entry == "robust_weight":
        got = O.robust_weight(d["f"], d["b"], 1.0, 0.1)
        np.testing.assert_allclose(got, d["out"], rtol=0, atol=1e-14)
        return
    if entry == "diffusion_term":
        np.testing.assert_allclose(O.diffusion(d["f"], float(d["eps"])), d["out"], rtol=0, atol=1e-12)
        assert O.diffusion_energy(d["f"], float(d["eps"])) == pytest.approx(float(d["energy"]), rel=1e-13)
        return
    psf = oracle_psf(d)
    if entry == "wiener_1d":
        got = O.wiener_1d(d["f"], psf, float(d["k"]))
    elif entry == "wiener_2d":
        got = O.wiener_2d(d["f"], psf, float(d["k"]))
    elif entry == "box_convolve":
        got = O.box_filter(d["f"], psf.length, psf.center, 0 if psf.axis == "v" else 1)
    elif entry == "spatial_convolve":
        got = O.clamped_convolve(d["f"], psf)
    elif entry == "fourier_convolve":
        got = O.periodic_convolve(d["f"], psf)
    elif entry == "rrrl_step":
        params = oracle_params(d)
        conv = O.make_convolver(psf, d["u"].shape, "box")
        b, w, df = O.prepare_state(d["u"], d["f"], conv, params)
        np.testing.assert_allclose(b, d["blurred"], rtol=0, atol=1e-10)
        np.testing.assert_allclose(w, d["weight"], rtol=0, atol=1e-14)
        np.testing.assert_allclose(df, d["diffusion"], rtol=0, atol=1e-10)
        got = O.rrrl_step(d["u"], d["f"], (b, w, df), conv, params)
    else:
        raise AssertionError(entry)
    np.testing.assert_allclose(got, d["out"], rtol=0, atol=1e-9)


def test_lut_interpolation_accuracy():
    """test_deconv.py:20-31 restated on the oracle's table."""
    lut = O.default_lut()
    xs = np.linspace(lut.delta, lut.upper, 200_001)
    got = O.r1(xs)
    mask = xs >= lut.direct_below
    assert np.abs(got[mask] - (xs[mask] - 1 - np.log(xs[mask]))).max() < 1e-4
    assert O.r1(np.array([1.0]))[0] == 0.0


def test_fft_matches_naive_dft(rng):
    """test_fft.py:53-58 restated."""
    p = O.plan(16)
    k = np.arange(16)
    dft = np.exp(-2j * np.pi * np.outer(k, k) / 16)
    for _ in range(20):
        x = rng.uniform(-255, 255, 16)
        np.testing.assert_allclose(p.forward(x), dft @ x, rtol=0, atol=1e-10)


def test_periodic_direct_equals_fourier_convolver(rng):
    """Direct wrap-around convolution equals the FFT convolvers (basis of kernel K4)."""
    a = rng.uniform(0, 255, (32, 64))
    p2 = O.make_psf("2d", rng.uniform(0, 1, (5, 7)), center=(1, 5))
    np.testing.assert_allclose(O.periodic_convolve(a, p2), O.make_convolver(p2, a.shape, "fourier").blur(a),
                               rtol=0, atol=1e-9)
    p1 = O.make_psf("1d", rng.uniform(0, 1, 9), center=2, axis="h")
    np.testing.assert_allclose(O.periodic_convolve(a, p1), O.make_convolver(p1, a.shape, "fourier").blur(a),
                               rtol=0, atol=1e-9)


# ---- drop-in boundary fixtures (oracle/gen_golden_boundary.py, produced by the reference)

LUT_ARGS = dict(delta=1.0 / 16.0, step=1.0 / 1000.0, upper=40.0, direct_below=0.4)


def test_oracle_custom_lut_golden():
    from oracle import wr3l_oracle as O
    d = load_golden("bnd_lut_custom")
    lut = O.build_lut(**LUT_ARGS)
    np.testing.assert_array_equal(lut.table, d["table"])
    np.testing.assert_allclose(O.r1(d["x"], lut), d["out"], rtol=0, atol=1e-15)


def test_oracle_custom_lut_pipelines_golden():
    from oracle import wr3l_oracle as O
    lut = O.build_lut(**LUT_ARGS)
    d = load_golden("bnd_pipe_lut_custom")
    got = O.pipeline(d["f"].astype(np.float64), O.make_psf("box", axis="h", length=9), O.OParams(), "box", lut=lut)
    assert np.abs(got - d["out"]).max() <= 1e-8
    d = load_golden("bnd_rrrl_lut_custom")
    spec = O.OPsf("1d", d["psf_weights"], int(d["psf_center"]), "v")
    conv = O.make_convolver(spec, d["f"].shape, "fourier")
    fpos = np.maximum(d["f"].astype(np.float64), 0.1)
    u = fpos.copy()
    for _ in range(4):
        u = O.rrrl_iteration(u, fpos, conv, O.OParams(iterations=4), lut)
    assert np.abs(u - d["out"]).max() <= 1e-8


def test_oracle_object_convolver_golden():
    from oracle import wr3l_oracle as O
    spec = O.make_psf("box", axis="h", length=9)
    conv = O.SpatialConv(O.OPsf("1d", spec.weights, spec.center, "h"))
    d = load_golden("bnd_rrrl_object")
    fpos = np.maximum(d["f"].astype(np.float64), 0.1)
    u = fpos.copy()
    for _ in range(5):
        u = O.rrrl_iteration(u, fpos, conv, O.OParams())
    assert np.abs(u - d["out"]).max() <= 1e-8
