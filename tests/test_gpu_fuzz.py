"""Seeded random sweep of the CUDA pipeline against the CPU oracle: PSF kind (box of integer /
even / fractional length, general 1D, 2D line, small dense 2D), blur axis, frame shape
(power-of-two axes as the FFT-based Wiener requires, square and not), parameters (K, alpha,
iterations, eps), noise level, the scenario (BOX_1D / FOURIER_1D / FOURIER_2D, including a 1D
PSF through the 2D scenario) and the dtype.
Each case is small so the NumPy oracle finishes in well under a second; the bar is the
north_star's max|d| <= 1e-4 * 255 (float64 everywhere; float32 only on the noisy cases where
SURVEY.md 7 measured it safe)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4 * 255.0
N_CASES = 120


@pytest.fixture(scope="module")
def md():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1212_2245_b200 as md
    return md


def _case(md, i):
    rng = np.random.default_rng(1000 + i)
    H = int(rng.choice([32, 64, 128, 256]))
    W = int(rng.choice([32, 64, 128, 256]))
    kind = ["box", "1d", "line", "dense"][i % 4]
    axis = md.BlurAxis.HORIZONTAL if rng.random() < 0.5 else md.BlurAxis.VERTICAL
    along = W if axis is md.BlurAxis.HORIZONTAL else H
    if kind == "box":
        L = float(rng.integers(2, min(31, along // 2)))
        if rng.random() < 0.4:
            L += 0.5
        psf = md.Psf.uniform_box(axis, L)
    elif kind == "1d":
        t = int(rng.integers(3, min(17, along // 2)))
        psf = md.Psf.general_1d(rng.uniform(0.1, 1.0, t), axis, center=int(rng.integers(0, t)))
    elif kind == "line":
        psf = md.Psf.line(float(rng.uniform(3.0, min(15.0, min(H, W) / 3))), float(rng.uniform(0.0, 180.0)))
    else:
        s = int(rng.integers(2, 6))
        psf = md.Psf.general_2d(rng.uniform(0.0, 1.0, (s, s)))
    params = md.DeconvParams(wiener_k=float(rng.uniform(0.002, 0.05)), alpha=float(rng.choice([0.0, 0.003, 0.01])),
                             iterations=int(rng.integers(0, 6)), eps_data=float(rng.choice([0.5, 1.0, 2.0])),
                             eps_reg=float(rng.choice([0.01, 0.05])))
    sigma = float(rng.choice([0.0, 2.0, 5.0]))
    g = md.make_test_image(W, H, seed=int(rng.integers(0, 100)))
    f = md.synth_blur(g, psf)
    if sigma > 0:
        f = md.quantize(md.add_gaussian_noise(f, sigma, seed=int(rng.integers(0, 1000))))
    if psf.kind is md.PsfKind.UNIFORM_BOX_1D:
        scen = [md.Scenario.BOX_1D, md.Scenario.FOURIER_1D, md.Scenario.FOURIER_2D][int(rng.integers(0, 3))]
    elif psf.kind is md.PsfKind.GENERAL_1D:
        scen = [md.Scenario.FOURIER_1D, md.Scenario.FOURIER_2D][int(rng.integers(0, 2))]
    else:
        scen = md.Scenario.FOURIER_2D
    return psf, params, f, sigma, scen


def _oracle(md, f, psf, params, scen):
    from oracle import wr3l_oracle as O
    ax = None if psf.axis is None else ("h" if psf.axis is md.BlurAxis.HORIZONTAL else "v")
    if psf.kind is md.PsfKind.UNIFORM_BOX_1D:
        op = O.make_psf("box", axis=ax, length=psf.length)
    elif psf.kind is md.PsfKind.GENERAL_1D:
        op = O.OPsf("1d", np.asarray(psf.weights), int(psf.center), ax)
    else:
        op = O.OPsf("2d", np.asarray(psf.weights), tuple(psf.center))
    p = O.OParams(params.wiener_k, params.alpha, params.iterations, params.eps_data, params.eps_reg, params.floor)
    return O.pipeline(f.values, op, p, scen.value)


@pytest.mark.parametrize("i", range(N_CASES))
def test_random_pipeline_vs_oracle(md, i):
    psf, params, f, sigma, scen = _case(md, i)
    ref = _oracle(md, f, psf, params, scen)
    out = md.DeblurPipeline(f.shape, psf, params, scen).run(f).values
    assert np.abs(out - ref).max() <= TOL, ("float64", i)
    if sigma >= 5.0 and psf.kind is not md.PsfKind.GENERAL_2D:
        out32 = md.DeblurPipeline(f.shape, psf, params, scen, dtype="float32").run(f).values
        assert np.abs(out32 - ref).max() <= TOL, ("float32", i)
