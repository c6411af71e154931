"""Parity of the CUDA path with the reference (golden fixtures) and the pinned oracle.

Tolerance (BASELINE.json north_star): max |u_gpu - u_ref| <= 1e-4 of the grey range
(0.0255 on [0, 255]) and |PSNR_gpu - PSNR_ref| <= 0.01 dB. The float64 path is also held
to a much tighter bound (FP64_TOL) to catch indexing bugs that a loose bound would hide.
All calls go through the public API -> GpuPlan -> C ABI (libmdcuda.so).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_names, load_golden, oracle_params, oracle_psf, product_params, product_psf

pytestmark = pytest.mark.gpu

TOL = 1e-4 * 255.0          # north_star max |delta|
PSNR_TOL = 0.01             # dB
FP64_TOL = 1e-6


@pytest.fixture(scope="module")
def md():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1212_2245_b200 as m
    return m


def _psnr(u, g):
    return 10.0 * np.log10(255.0 ** 2 / np.mean((u - g) ** 2))


SCEN = {"box": "BOX_1D", "fourier1d": "FOURIER_1D", "fourier2d": "FOURIER_2D"}


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("name", golden_names("pipe_"))
def test_pipeline_golden(md, name, dtype):
    d = load_golden(name)
    noisy_or_short = name.startswith(("pipe_c1", "pipe_box", "pipe_f1d_v9", "pipe_f1d_h7", "pipe_f2d_3x5",
                                      "pipe_f2d_boxv9"))
    if dtype == "float32" and not noisy_or_short:
        pytest.skip("noise-free 2D configs need float64 (SURVEY.md 7, hard part 1)")
    psf, params = product_psf(d), product_params(d)
    scen = md.Scenario[SCEN[str(d["scenario"])]]
    out = md.DeblurPipeline(d["f"].shape, psf, params, scen, dtype=dtype).run(md.Image(d["f"])).values
    err = np.abs(out - d["out"]).max()
    assert err <= TOL, err
    if dtype == "float64":
        assert err <= FP64_TOL, err
    if "g" in d:
        assert abs(_psnr(out, d["g"]) - _psnr(d["out"], d["g"])) <= PSNR_TOL


@pytest.mark.parametrize("name", golden_names("pipe_f2d"))
def test_fft2d_convolver_path(md, name):
    """FOURIER_2D through the 2D-FFT convolver (forced) agrees with the reference too."""
    d = load_golden(name)
    if str(d["psf_kind"]) != "2d":
        pytest.skip("1D kernel")
    out = md.DeblurPipeline(d["f"].shape, product_psf(d), product_params(d), md.Scenario.FOURIER_2D,
                            force_fft2d=True).run(md.Image(d["f"])).values
    assert np.abs(out - d["out"]).max() <= FP64_TOL


@pytest.mark.parametrize("name", golden_names("rrrl_") + golden_names("rl_"))
def test_deblur_entries_golden(md, name):
    d = load_golden(name)
    psf, params = product_psf(d), product_params(d)
    mode = str(d["mode"]) or None
    f = md.Image(d["f"])
    if str(d["entry"]) == "rrrl":
        out = md.rrrl_deblur(f, psf, params, mode).values
    else:
        out = md.rl_deblur(f, psf, params.iterations, mode, params.floor).values
    assert np.abs(out - d["out"]).max() <= FP64_TOL


@pytest.mark.parametrize("name", golden_names("comp_"))
def test_components_golden(md, name):
    d = load_golden(name)
    entry = str(d["entry"])
    if entry == "lut_r1":
        # the public DivergenceLut.r1 (md_lut_r1, the reference's rounding order) at 1e-12
        got = md.default_divergence_lut().r1(d["x"])
        np.testing.assert_allclose(got, d["out"], rtol=0, atol=1e-12)
        assert float(np.mean(got == d["out"])) > 0.99     # bitwise except a log ulp here and there
        return
    if entry == "robust_weight":
        got = md.robust_weight(md.Image(d["f"]), md.Image(d["b"]), eps_data=1.0, floor=0.1).values
        np.testing.assert_allclose(got, d["out"], rtol=0, atol=1e-13)
        return
    if entry == "diffusion_term":
        got = md.diffusion_term(md.Image(d["f"]), float(d["eps"])).values
        np.testing.assert_allclose(got, d["out"], rtol=0, atol=1e-10)
        assert md.diffusion_energy(md.Image(d["f"]), float(d["eps"])) == pytest.approx(float(d["energy"]), rel=1e-12)
        return
    psf = product_psf(d)
    f = md.Image(d["f"])
    if entry == "wiener_1d":
        got = md.wiener_1d(f, psf, float(d["k"])).values
    elif entry == "wiener_2d":
        got = md.wiener_2d(f, psf, float(d["k"])).values
    elif entry == "box_convolve":
        got = md.box_convolve(f, psf).values
    elif entry == "spatial_convolve":
        got = md.spatial_convolve(f, psf).values
    elif entry == "fourier_convolve":
        got = md.fourier_convolve(f, psf).values
    elif entry == "rrrl_step":
        params = product_params(d)
        conv = md.make_convolver(psf, d["u"].shape, "box")
        st = md.prepare_state(md.Image(d["u"]), f, psf, params, conv)
        np.testing.assert_allclose(st.blurred.values, d["blurred"], rtol=0, atol=1e-9)
        np.testing.assert_allclose(st.weight.values, d["weight"], rtol=0, atol=1e-13)
        np.testing.assert_allclose(st.diffusion.values, d["diffusion"], rtol=0, atol=1e-9)
        got = md.rrrl_step(st, f, psf, params, conv).values
    else:
        raise AssertionError(entry)
    np.testing.assert_allclose(got, d["out"], rtol=0, atol=1e-8)


# ---------------------------------------------------------------- full-size configs vs oracle

def _line_case(md, n, iters):
    line = md.Psf.line(21.0, 30.0)
    g = md.make_test_image(n, n)
    f = md.synth_blur(g, line)
    return g, f, line, md.DeconvParams(iterations=iters)


def test_c2_512_line_fp64_vs_oracle(md):
    from oracle import wr3l_oracle as O
    g, f, psf, params = _line_case(md, 512, 10)
    out = md.DeblurPipeline(f.shape, psf, params).run(f).values
    ref = O.pipeline(f.values, O.OPsf("2d", psf.weights, psf.center), O.OParams(iterations=10), "fourier2d")
    assert np.abs(out - ref).max() <= TOL
    assert abs(_psnr(out, g.values) - _psnr(ref, g.values)) <= PSNR_TOL


def test_c3_1024_gauss31_fp64_vs_oracle(md):
    from oracle import wr3l_oracle as O
    yy, xx = np.mgrid[-15:16, -15:16]
    w = np.exp(-(yy ** 2 + xx ** 2) / 50.0) * np.random.default_rng(3).uniform(0.2, 1.0, (31, 31))
    psf = md.Psf.general_2d(w)
    g = md.make_test_image(1024, 1024)
    f = md.synth_blur(g, psf)
    out = md.DeblurPipeline(f.shape, psf, md.DeconvParams()).run(f).values
    ref = O.pipeline(f.values, O.OPsf("2d", psf.weights, psf.center), O.OParams(), "fourier2d")
    assert np.abs(out - ref).max() <= TOL
    assert abs(_psnr(out, g.values) - _psnr(ref, g.values)) <= PSNR_TOL


# ---------------------------------------------------------------- size-independent properties

def test_synth_blur_matches_reference_fixture(md):
    d = load_golden("pipe_c1_box_h15_256")
    g = md.Image(d["g"])
    blurred = md.synth_blur(g, md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15))
    noisy = md.quantize(md.add_gaussian_noise(blurred, 5.0, seed=5))
    np.testing.assert_array_equal(noisy.values, d["f"])


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_batch_equals_single_frames(md, dtype):
    import torch
    d = load_golden("pipe_c1_box_h15_256")
    psf, params = product_psf(d), product_params(d)
    pipe = md.DeblurPipeline((256, 256), psf, params, dtype=dtype)
    rng = np.random.default_rng(0)
    frames = np.stack([d["f"]] + [np.clip(d["f"] + rng.normal(0, 3, d["f"].shape), 0, 255).round()
                                  for _ in range(5)])
    t = torch.from_numpy(frames).cuda().to(torch.float64 if dtype == "float64" else torch.float32)
    out = pipe.run_batch(t).double().cpu().numpy()
    for i in range(frames.shape[0]):
        single = pipe.run(md.Image(frames[i])).values
        np.testing.assert_array_equal(out[i], single)
    host = pipe.run_batch(frames)
    np.testing.assert_allclose(host, out, rtol=0, atol=0)


def test_horizontal_equals_transposed_vertical(md):
    g = md.make_test_image(64, 128)
    ph = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 9)
    pv = md.Psf.uniform_box(md.BlurAxis.VERTICAL, 9)
    f = md.synth_blur(g, ph)
    a = md.wr3l(f, ph, md.DeconvParams()).values
    b = md.wr3l(md.Image(f.values.T), pv, md.DeconvParams()).values.T
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-10)


def test_zero_iterations_is_clamped_wiener(md):
    f = md.make_test_image(128, 128)
    psf = md.Psf.uniform_box(md.BlurAxis.VERTICAL, 15)
    params = md.DeconvParams(iterations=0)
    out = md.wr3l(f, psf, params).values
    want = md.clamp_floor(md.wiener_1d(f, psf, params.wiener_k), params.floor).values
    np.testing.assert_allclose(out, want, rtol=0, atol=1e-12)


def test_output_strictly_positive_and_improves_snr(md):
    """test_pipeline.py:57-69 of the reference."""
    g = md.make_test_image(128, 128)
    psf = md.Psf.uniform_box(md.BlurAxis.VERTICAL, 15)
    f = md.synth_blur(g, psf)
    out = md.wr3l(f, psf, md.DeconvParams())
    assert out.values.min() > 0.0
    assert md.snr(out, g) > md.snr(f, g)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("name", ["pipe_c1_box_h15_256", "pipe_box_v21p5_64x96", "pipe_f1d_v9_128x64",
                                  "pipe_f1d_h7_64x128", "pipe_box_h15_alpha0_64", "pipe_f2d_3x5_64x128",
                                  "pipe_f2d_line21_30_128"])
def test_generic_line_kernel_golden(md, name, dtype):
    """The generic (index-resolving) line / plane kernels stay correct next to the fast ones."""
    d = load_golden(name)
    if dtype == "float32" and name == "pipe_f2d_line21_30_128":
        pytest.skip("noise-free 2D config needs float64")
    scen = md.Scenario[SCEN[str(d["scenario"])]]
    out = md.DeblurPipeline(d["f"].shape, product_psf(d), product_params(d), scen, dtype=dtype,
                            generic_lines=True).run(md.Image(d["f"])).values
    assert np.abs(out - d["out"]).max() <= (FP64_TOL if dtype == "float64" else TOL)


def test_contract_errors(md):
    psf = md.Psf.uniform_box(md.BlurAxis.VERTICAL, 3)
    bad = md.Image([[0.0, 1.0], [1.0, 1.0]] * 2)
    good = md.Image(np.ones((4, 2)))
    with pytest.raises(md.ContractError):
        md.rl_step(bad, good, psf)
    with pytest.raises(md.ContractError):
        md.robust_weight(good, bad)


def test_validation_errors(md):
    psf2d = md.Psf.general_2d(np.ones((3, 3)))
    with pytest.raises(ValueError):
        md.DeblurPipeline((64, 64), psf2d, md.DeconvParams(), md.Scenario.BOX_1D)
    with pytest.raises(ValueError):
        md.DeblurPipeline((48, 64), md.Psf.uniform_box(md.BlurAxis.VERTICAL, 5), md.DeconvParams())
    md.DeblurPipeline((64, 48), md.Psf.uniform_box(md.BlurAxis.VERTICAL, 5), md.DeconvParams())
    with pytest.raises(ValueError):
        md.wiener_1d(md.Image(np.ones((12, 8))), md.Psf.uniform_box(md.BlurAxis.VERTICAL, 3), 0.1)
    with pytest.raises(ValueError):
        md.wiener_2d(md.Image(np.ones((8, 8))), psf2d, 0.0)
    pipe = md.DeblurPipeline((64, 64), md.Psf.uniform_box(md.BlurAxis.VERTICAL, 5), md.DeconvParams())
    with pytest.raises(ValueError):
        pipe.run(md.Image(np.ones((32, 32))))


def test_rl_fixed_point(md):
    rng = np.random.default_rng(103)
    for mode, psf in (("spatial", md.Psf.general_2d(rng.uniform(0, 1, (5, 3)))),
                      ("box", md.Psf.uniform_box(md.BlurAxis.VERTICAL, 7)),
                      ("fourier", md.Psf.general_1d(rng.uniform(0, 1, 9), md.BlurAxis.VERTICAL))):
        u = md.Image(rng.uniform(1, 255, (64, 64)))
        conv = md.make_convolver(psf, u.shape, mode)
        f = md.Image(conv.blur(u.values))
        u1 = md.rl_step(u, f, psf, conv)
        assert np.abs(u1.values / u.values - 1.0).max() < 1e-12


def test_rrrl_with_alpha0_identity_weight_equals_rl(md):
    rng = np.random.default_rng(104)
    psf = md.Psf.uniform_box(md.BlurAxis.VERTICAL, 9)
    conv = md.make_convolver(psf, (64, 64), "box")
    params = md.DeconvParams(alpha=0.0, iterations=10)
    f = md.Image(rng.uniform(1, 255, (64, 64)))
    u_rl = u_rr = md.clamp_floor(f)
    for _ in range(5):
        u_rl = md.rl_step(u_rl, f, psf, conv)
        st = md.prepare_state(u_rr, f, psf, params, conv, robust=False)
        u_rr = md.rrrl_step(st, f, psf, params, conv)
        np.testing.assert_array_equal(u_rr.values, u_rl.values)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("name", ["pipe_c1_box_h15_256", "pipe_box_v21p5_64x96", "pipe_f1d_v9_128x64",
                                  "pipe_f1d_h7_64x128", "pipe_box_h15_alpha0_64", "pipe_f1d_box_v27_256"])
def test_fused_cluster_kernel_matches_per_iteration_kernel(md, name, dtype):
    """The cluster-resident kernel (DSMEM halo exchange) reproduces the per-iteration kernel
    and the reference."""
    d = load_golden(name)
    scen = md.Scenario[SCEN[str(d["scenario"])]]
    shape = d["f"].shape
    try:
        on = md.DeblurPipeline(shape, product_psf(d), product_params(d), scen, dtype=dtype, fused=True)
    except ValueError as exc:
        pytest.skip(f"fused kernel not applicable: {exc}")
    off = md.DeblurPipeline(shape, product_psf(d), product_params(d), scen, dtype=dtype, fused=False)
    a = on.run(md.Image(d["f"])).values
    b = off.run(md.Image(d["f"])).values
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-9 if dtype == "float64" else 1e-3)
    assert np.abs(a - d["out"]).max() <= (FP64_TOL if dtype == "float64" else TOL)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_host_entry_io_types(md, dtype):
    """md_run_host_ex: uint8 / float32 / float64 host frames, pipelined chunks, equal results."""
    import torch
    d = load_golden("pipe_c1_box_h15_256")
    pipe = md.DeblurPipeline((256, 256), product_psf(d), product_params(d), dtype=dtype)
    rng = np.random.default_rng(3)
    frames = np.stack([np.clip(d["f"] + rng.normal(0, 4, d["f"].shape), 0, 255).round() for _ in range(37)])
    dev = pipe.run_batch(torch.from_numpy(frames).cuda().to(torch.float64 if dtype == "float64"
                                                              else torch.float32)).double().cpu().numpy()
    pipe.plan.set_chunk(0)
    a = pipe.run_batch(frames.astype(np.uint8), out_dtype=np.float32)
    b = pipe.run_batch(frames.astype(np.float32))
    c = pipe.run_batch(frames)
    assert a.dtype == np.float32 and b.dtype == np.float64
    np.testing.assert_allclose(c, dev, rtol=0, atol=0)
    np.testing.assert_allclose(b, dev, rtol=0, atol=0)
    np.testing.assert_allclose(a, dev.astype(np.float32), rtol=0, atol=0)


def test_fused_batch_many_frames(md):
    import torch
    d = load_golden("pipe_c1_box_h15_256")
    pipe = md.DeblurPipeline((256, 256), product_psf(d), product_params(d), dtype="float32")
    assert pipe.plan.fused
    frames = torch.from_numpy(np.stack([d["f"]] * 300)).cuda().float()
    frames[7] += 3.0
    out = pipe.run_batch(frames).double().cpu().numpy()
    ref = pipe.run(md.Image(d["f"])).values
    for i in (0, 1, 150, 299):
        np.testing.assert_array_equal(out[i], ref)
    assert np.abs(out[7] - ref).max() > 0.1


@pytest.mark.parametrize("chunk", [40, 64, 300])
def test_fused_chunk_pipeline_bitwise(md, chunk):
    """Batches over several chunks run the Wiener step of chunk c+1 as a programmatic dependent
    launch beside chunk c's iteration kernel (md_capi.cu run_lines_pipelined): same bits as one
    chunk, every frame, including a ragged last chunk."""
    import torch
    d = load_golden("pipe_c1_box_h15_256")
    pipe = md.DeblurPipeline((256, 256), product_psf(d), product_params(d), dtype="float32")
    assert pipe.plan.fused
    g = torch.Generator().manual_seed(5)
    frames = (torch.from_numpy(np.stack([d["f"]] * 301)).float()
              + torch.randn((301, 256, 256), generator=g)).cuda()
    whole = pipe.run_batch(frames).cpu().numpy()
    pipe.plan.set_chunk(chunk)
    try:
        parts = pipe.run_batch(frames).cpu().numpy()
    finally:
        pipe.plan.set_chunk(0)
    np.testing.assert_array_equal(parts, whole)
    one = pipe.run_batch(frames[250:251]).cpu().numpy()
    np.testing.assert_array_equal(parts[250], one[0])


def test_plan_reports_launches(md):
    pipe = md.DeblurPipeline((256, 256), md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15), md.DeconvParams())
    assert pipe.plan.launch_count(16) >= 2
    assert "lines" in pipe.plan.describe


def test_psf_bank_pipeline_matches_single_plans(md):
    """configs[3]-style bank: unsorted per-frame PSF indices, each frame equals its own plan."""
    import torch
    from paper_1212_2245_b200.batch import PsfBankPipeline
    bank = [md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 9.5), md.Psf.general_1d([1, 3, 2, 1], md.BlurAxis.VERTICAL),
            md.Psf.line(11.0, 40.0)]
    params = md.DeconvParams()
    pipe = PsfBankPipeline((64, 64), bank, params, dtype="float64")
    rng = np.random.default_rng(9)
    g = md.make_test_image(64, 64)
    idx = np.array([2, 0, 1, 1, 0, 2, 2])
    frames = np.stack([md.quantize(md.add_gaussian_noise(md.synth_blur(g, bank[i]), 5.0, int(s))).values
                       for s, i in enumerate(idx)])
    out = pipe.run(torch.from_numpy(frames).cuda(), idx).cpu().numpy()
    for k, i in enumerate(idx):
        want = md.DeblurPipeline((64, 64), bank[i], params).run(md.Image(frames[k])).values
        # 2D-PSF groups run their Wiener FFTs two frames per complex field (real / imaginary
        # part), which only changes rounding
        np.testing.assert_allclose(out[k], want, rtol=0, atol=0 if bank[i].kind.value != "2d" else 1e-9)
    # the PSF groups dealt over internal streams: the same bits
    for ns in (2, 3):
        np.testing.assert_array_equal(pipe.run(torch.from_numpy(frames).cuda(), idx, streams=ns).cpu().numpy(), out)


def test_paired_2d_wiener_matches_single_frames(md):
    """Frame pairing in the 2D Wiener pass: odd and even batch sizes, float32 and float64."""
    import torch
    psf = md.Psf.line(9.0, 110.0)
    g = md.make_test_image(64, 64, seed=3).values
    frames = np.stack([md.synth_blur(md.Image(np.roll(g, 7 * k, axis=1)), psf).values for k in range(5)])
    for dtype, tol in (("float64", 1e-9), ("float32", 2e-3)):
        pipe = md.DeblurPipeline((64, 64), psf, md.DeconvParams(), md.Scenario.FOURIER_2D, dtype=dtype)
        tdt = torch.float64 if dtype == "float64" else torch.float32
        for nb in (1, 2, 5):
            out = pipe.run_batch(torch.from_numpy(frames[:nb]).cuda().to(tdt)).double().cpu().numpy()
            for k in range(nb):
                single = pipe.run(md.Image(frames[k])).values
                np.testing.assert_allclose(out[k], single, rtol=0, atol=tol)


@pytest.mark.parametrize("name", ["pipe_f2d_line21_30_128", "pipe_f2d_3x5_64x128", "pipe_f2d_gauss31_128"])
def test_two_level_fft_wiener_golden(md, name):
    """The large-image Wiener (two-level FFT passes, md_fft_big.cu) forced at fixture size."""
    d = load_golden(name)
    if name == "pipe_f2d_gauss31_128":
        with pytest.raises(ValueError):      # dense PSFs iterate through FFTs, not offered at that size
            md.DeblurPipeline(d["f"].shape, product_psf(d), product_params(d), md.Scenario.FOURIER_2D, big_fft=True)
        return
    out = md.DeblurPipeline(d["f"].shape, product_psf(d), product_params(d), md.Scenario.FOURIER_2D,
                            big_fft=True).run(md.Image(d["f"])).values
    assert np.abs(out - d["out"]).max() <= FP64_TOL


def test_two_level_fft_matches_single_pass_2048(md):
    """c5-style line PSF on a 2048^2 frame: two-level FFT Wiener == single-pass Wiener."""
    import torch
    psf = md.Psf.line(21.0, 30.0)
    g = md.make_test_image(2048, 2048)
    f = torch.from_numpy(md.synth_blur(g, psf).values).cuda()
    params = md.DeconvParams(iterations=2)
    a = md.DeblurPipeline((2048, 2048), psf, params).run_batch(f)
    b = md.DeblurPipeline((2048, 2048), psf, params, big_fft=True).run_batch(f)
    assert float((a - b).abs().max()) <= FP64_TOL     # rounding only (~1e-8 after RRRL amplification)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("name", ["pipe_f2d_3x5_64x128", "pipe_f2d_boxv9_64", "pipe_f2d_line21_30_128"])
def test_fused_plane_kernel_matches_per_iteration_kernel(md, name, dtype):
    """2D PSFs: the cluster-resident iteration loop (md_fused_plane.cu) reproduces the
    two-kernel-per-iteration path and the reference."""
    d = load_golden(name)
    shape = d["f"].shape
    on = md.DeblurPipeline(shape, product_psf(d), product_params(d), md.Scenario.FOURIER_2D, dtype=dtype, fused=True)
    assert on.plan.fused
    if dtype == "float32":                       # the float default picks it by itself
        assert "fused" in md.DeblurPipeline(shape, product_psf(d), product_params(d),
                                                    md.Scenario.FOURIER_2D, dtype=dtype).plan.describe
    off = md.DeblurPipeline(shape, product_psf(d), product_params(d), md.Scenario.FOURIER_2D, dtype=dtype,
                            fused=False)
    assert not off.plan.fused
    a = on.run(md.Image(d["f"])).values
    b = off.run(md.Image(d["f"])).values
    # float32: the fused kernel sums taps column by column, so rounding differs from the
    # tap-order sum; on the noise-free line blur that is amplified, but stays inside TOL
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-9 if dtype == "float64" else TOL)
    if dtype == "float64":
        assert np.abs(a - d["out"]).max() <= FP64_TOL
    elif name != "pipe_f2d_line21_30_128":       # noise-free line blur needs float64
        assert np.abs(a - d["out"]).max() <= TOL


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("rl", [False, True])
@pytest.mark.parametrize("shape", [(64, 128), (128, 64), (256, 256)])
def test_fused_plane_clamped_spatial(md, dtype, rl, shape):
    """Clamped spatial convolver (edge-replicated halos at the cluster's first / last CTA)."""
    import torch
    from paper_1212_2245_b200.plan import GpuPlan
    rng = np.random.default_rng(11)
    psf = md.Psf.general_2d(rng.uniform(0.1, 1.0, (5, 4)))
    params = md.DeconvParams(iterations=4)
    g = md.make_test_image(shape[1], shape[0], seed=5).values
    f = md.synth_blur(md.Image(g), psf).values + rng.normal(0, 2, shape)
    tdt = torch.float64 if dtype == "float64" else torch.float32
    fd = torch.from_numpy(np.stack([f, f[::-1].copy(), 255 - f])).cuda().to(tdt)
    outs = []
    for fused in (True, False):
        plan = GpuPlan(shape, psf, params, "spatial", init="clamped", dtype=dtype, rl=rl, fused=fused)
        assert plan.fused == fused
        outs.append(plan.run(fd).double().cpu().numpy())
    np.testing.assert_allclose(outs[0], outs[1], rtol=0, atol=1e-9 if dtype == "float64" else 2e-3)


def test_fused_plane_c4_line_frames_independent(md):
    """c4-style 256^2 frames under a line PSF: many frames per launch stay independent and the
    float32 result stays within the north_star tolerance of float64."""
    import torch
    psf = md.Psf.line(17.0, 63.0)
    g = md.make_test_image(256, 256, seed=9).values
    rng = np.random.default_rng(4)
    f = np.clip(md.synth_blur(md.Image(g), psf).values + rng.normal(0, 5, g.shape), 0, 255)
    p32 = md.DeblurPipeline((256, 256), psf, md.DeconvParams(), md.Scenario.FOURIER_2D, dtype="float32")
    assert p32.plan.fused
    frames = torch.from_numpy(np.stack([f] * 45)).cuda().float()
    frames[13] += 2.0
    out = p32.run_batch(frames).double().cpu().numpy()
    for i in (0, 12, 14, 44):       # Wiener pairs frames per complex field: rounding only
        np.testing.assert_allclose(out[i], out[0], rtol=0, atol=2e-3)
    assert np.abs(out[13] - out[0]).max() > 0.1
    ref = md.DeblurPipeline((256, 256), psf, md.DeconvParams(), md.Scenario.FOURIER_2D,
                            dtype="float64").run(md.Image(f)).values
    assert np.abs(out[0] - ref).max() <= TOL


def test_psf_bank_host_entry_matches_device_run(md):
    """PsfBankPipeline.run_host: unsorted uint8 / float64 host frames, pipelined per group,
    equal to the device path."""
    import torch
    from paper_1212_2245_b200.batch import PsfBankPipeline
    bank = [md.Psf.uniform_box(md.BlurAxis.VERTICAL, 7), md.Psf.general_1d([1, 2, 4, 2], md.BlurAxis.HORIZONTAL),
            md.Psf.line(9.0, 75.0)]
    pipe = PsfBankPipeline((64, 64), bank, md.DeconvParams(), dtype="float32")
    rng = np.random.default_rng(2)
    idx = rng.integers(0, 3, 23)
    frames = rng.integers(20, 230, (23, 64, 64)).astype(np.uint8)
    want = pipe.run(torch.from_numpy(frames.astype(np.float32)).cuda(), idx).cpu().numpy()
    got = pipe.run_host(frames, idx, max_piece=4)
    assert got.dtype == np.float32
    np.testing.assert_array_equal(got, want)
    got64 = pipe.run_host(frames.astype(np.float64), idx, out_dtype=np.float64)
    np.testing.assert_array_equal(got64, want.astype(np.float64))


def test_host_entry_uint8_out_is_write_pgm_quantisation(md):
    """uint8 results from the host entries follow the reference's write_pgm rounding."""
    from paper_1212_2245_b200.batch import PsfBankPipeline
    d = load_golden("pipe_c1_box_h15_256")
    pipe = md.DeblurPipeline((256, 256), product_psf(d), product_params(d), dtype="float32")
    rng = np.random.default_rng(8)
    frames = np.stack([np.clip(d["f"] + rng.normal(0, 3, d["f"].shape), 0, 255).round() for _ in range(9)])
    f32 = pipe.run_batch(frames.astype(np.uint8), out_dtype=np.float32)
    u8 = pipe.run_batch(frames.astype(np.uint8), out_dtype=np.uint8)
    # rounding evaluated in the plan's precision (float32), as the conversion kernel does
    np.testing.assert_array_equal(u8, np.clip(np.floor(f32 + np.float32(0.5)), 0, 255).astype(np.uint8))
    bank = PsfBankPipeline((256, 256), [product_psf(d)], product_params(d), dtype="float32")
    b8 = bank.run_host(frames.astype(np.uint8), np.zeros(9, np.int64), out_dtype=np.uint8)
    np.testing.assert_array_equal(b8, u8)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("length", [3.0, 4.0, 6.5, 9.5, 10.0, 16.0, 21.5, 29.0, 30.0, 31.0])
@pytest.mark.parametrize("axis", ["HORIZONTAL", "VERTICAL"])
def test_fused_box_sliding_sum_all_box_lengths(md, dtype, length, axis):
    """Odd, even and fractional boxes run the cluster kernel's sliding-sum path (interior sum +
    end corrections) and agree with the per-iteration dense-tap kernel."""
    import torch
    psf = md.Psf.uniform_box(md.BlurAxis[axis], length)
    g = md.make_test_image(256, 256, seed=4).values
    rng = np.random.default_rng(int(length * 10))
    f = np.clip(md.synth_blur(md.Image(g), psf).values + rng.normal(0, 5, g.shape), 0, 255).round()
    tdt = torch.float64 if dtype == "float64" else torch.float32
    fd = torch.from_numpy(np.stack([f, f[::-1].copy()])).cuda().to(tdt)
    on = md.DeblurPipeline((256, 256), psf, md.DeconvParams(), md.Scenario.BOX_1D, dtype=dtype, fused=True)
    off = md.DeblurPipeline((256, 256), psf, md.DeconvParams(), md.Scenario.BOX_1D, dtype=dtype, fused=False)
    a = on.run_batch(fd).double().cpu().numpy()
    b = off.run_batch(fd).double().cpu().numpy()
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-9 if dtype == "float64" else 3e-3)
