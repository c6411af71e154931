"""The float64 cluster-resident iteration kernel (md_fused64_kernel.cuh: shuffle windows,
st.async halo lines, mbarrier-tracked exchange) against the CPU oracle, over the shapes and
convolvers it covers: box radii 1..8 (odd, even and fractional lengths), dense line taps
(FOURIER_1D: periodic), both blur axes, 2..16 CTAs per cluster (32..256 lines), lines of 64..256
samples, alpha = 0 (no diffusivity) and iteration counts 0..6. Bar: max|d| <= 1e-6 (float64;
north_star allows 1e-4 * 255). Also: the kernel is the default float64 path for these plans, a
batch equals its frames run one by one (bitwise), and it agrees with the per-iteration kernel."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def md():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1212_2245_b200 as md
    return md


def _oracle(md, f, psf, params, scen):
    from oracle import wr3l_oracle as O
    ax = "h" if psf.axis is md.BlurAxis.HORIZONTAL else "v"
    if psf.kind is md.PsfKind.UNIFORM_BOX_1D:
        op = O.make_psf("box", axis=ax, length=psf.length)
    else:
        op = O.OPsf("1d", np.asarray(psf.weights), int(psf.center), ax)
    p = O.OParams(params.wiener_k, params.alpha, params.iterations, params.eps_data, params.eps_reg, params.floor)
    return O.pipeline(f.values, op, p, scen.value)


CASES = [
    # (H, W, kind, length/taps, axis, alpha, iterations)
    (256, 256, "box", 15.0, "h", 0.003, 5),       # c1
    (256, 256, "box", 15.0, "v", 0.003, 5),
    (128, 128, "box", 3.0, "h", 0.003, 4),
    (64, 256, "box", 4.0, "h", 0.01, 3),          # even length
    (256, 64, "box", 9.5, "v", 0.003, 3),         # fractional
    (256, 128, "box", 17.0, "h", 0.003, 2),       # radius 8
    (32, 256, "box", 2.5, "h", 0.003, 6),         # two CTAs per cluster
    (256, 256, "box", 7.0, "h", 0.0, 5),          # no diffusion term
    (128, 256, "box", 11.0, "h", 0.003, 0),       # Wiener only
    (256, 256, "box", 13.0, "h", 0.003, 1),
    (256, 256, "taps", 7, "h", 0.003, 4),         # dense taps, periodic (FOURIER_1D)
    (128, 64, "taps", 9, "v", 0.01, 3),
    (64, 128, "taps", 5, "h", 0.0, 2),
    (256, 256, "box", 31.0, "h", 0.003, 5),       # radius 15: windows span two neighbour lanes
    (256, 256, "box", 21.5, "v", 0.003, 4),       # fractional, radius 11
    (128, 256, "box", 18.0, "h", 0.01, 3),        # even, radius 9
    (256, 128, "box", 33.0, "h", 0.003, 2),       # radius 16
    (256, 256, "taps", 17, "h", 0.003, 3),        # dense taps, radius 11 (centre 5)
    (64, 256, "taps", 29, "v", 0.003, 2),         # dense taps, radius 19 -> per-iteration kernel
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}-{c[2]}{c[3]}{c[4]}-a{c[5]}-it{c[6]}" for c in CASES])
def test_fused64_vs_oracle(md, case):
    H, W, kind, L, ax, alpha, its = case
    axis = md.BlurAxis.HORIZONTAL if ax == "h" else md.BlurAxis.VERTICAL
    rng = np.random.default_rng(H * 7 + W + its)
    if kind == "box":
        psf = md.Psf.uniform_box(axis, L)
        scen = md.Scenario.BOX_1D
    else:
        psf = md.Psf.general_1d(rng.uniform(0.1, 1.0, int(L)), axis, center=int(L) // 3)
        scen = md.Scenario.FOURIER_1D
    params = md.DeconvParams(alpha=alpha, iterations=its)
    g = md.make_test_image(W, H, seed=3)
    f = md.quantize(md.add_gaussian_noise(md.synth_blur(g, psf), 5.0, seed=11))
    pipe = md.DeblurPipeline(f.shape, psf, params, scen, dtype="float64")
    radius = max(int(L) // 2 + (1 if kind == "box" and L != int(L) else 0), 0) if kind == "box" else \
        max(int(L) // 3, int(L) - 1 - int(L) // 3)
    if its > 0 and radius <= 16:
        assert pipe.plan.fused, pipe.plan.describe
    out = pipe.run(f).values
    ref = _oracle(md, f, psf, params, scen)
    err = float(np.abs(out - ref).max())
    assert err <= 1e-6, err


def test_fused64_batch_is_framewise(md):
    import torch
    psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15)
    pipe = md.DeblurPipeline((256, 256), psf, md.DeconvParams(), md.Scenario.BOX_1D, dtype="float64")
    g = md.make_test_image(256, 256)
    b = md.synth_blur(g, psf).values
    frames = np.stack([np.clip(np.floor(b + np.random.default_rng(s).normal(0, 5, b.shape) + 0.5), 0, 255)
                       for s in range(37)])
    f = torch.from_numpy(frames).cuda()
    out = pipe.plan.run(f).cpu().numpy()
    for i in (0, 17, 36):
        one = pipe.plan.run(f[i:i + 1].contiguous()).cpu().numpy()[0]
        assert np.array_equal(one, out[i])


def test_fused64_matches_per_iteration_kernel(md):
    import torch
    psf = md.Psf.uniform_box(md.BlurAxis.VERTICAL, 15)
    params = md.DeconvParams()
    fused = md.DeblurPipeline((256, 256), psf, params, md.Scenario.BOX_1D, dtype="float64")
    plain = md.DeblurPipeline((256, 256), psf, params, md.Scenario.BOX_1D, dtype="float64", fused=False)
    assert fused.plan.fused and not plain.plan.fused
    g = md.make_test_image(256, 256, seed=9)
    f = md.quantize(md.add_gaussian_noise(md.synth_blur(g, psf), 5.0, seed=2))
    a, b = fused.run(f).values, plain.run(f).values
    assert float(np.abs(a - b).max()) <= 1e-9


@pytest.mark.parametrize("psf_kind", ["box15", "box21.5", "gen1d"])
def test_fused64_raw_observation_bitwise(md, psf_kind):
    """Horizontal lines run the cluster kernel on the raw observation (floored on load, no fpos
    field); vertical lines keep the transposing Wiener's fpos field. Same arithmetic either way:
    the horizontal result equals the transposed vertical one bit for bit."""
    ax_h, ax_v = md.BlurAxis.HORIZONTAL, md.BlurAxis.VERTICAL
    if psf_kind == "gen1d":
        w = np.exp(-0.5 * ((np.arange(13) - 6) / 2.5) ** 2)
        ph, pv = md.Psf.general_1d(w, ax_h), md.Psf.general_1d(w, ax_v)
    else:
        L = 15.0 if psf_kind == "box15" else 21.5
        ph, pv = md.Psf.uniform_box(ax_h, L), md.Psf.uniform_box(ax_v, L)
    g = md.make_test_image(256, 256, seed=4)
    f = md.quantize(md.add_gaussian_noise(md.synth_blur(g, ph), 5.0, seed=6))
    dh = md.DeblurPipeline((256, 256), ph, md.DeconvParams(), dtype="float64")
    dv = md.DeblurPipeline((256, 256), pv, md.DeconvParams(), dtype="float64")
    assert dh.plan.fused and dv.plan.fused
    a = dh.run(f).values
    b = dv.run(md.Image(np.ascontiguousarray(f.values.T))).values.T
    assert np.array_equal(a, b)
