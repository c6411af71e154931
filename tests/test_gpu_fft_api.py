"""The reference's transform API on the device (paper_1212_2245_b200/fft.py, md_fft) and
``rrrl_deblur_parallel``, against the CPU oracle's restatement of the reference FFT
(oracle/wr3l_oracle.py Radix2, pinned to the reference by tests/test_oracle_golden.py) and the
reference's own test properties (test_fft.py: naive DFT within 1e-10, periodic convolution)."""

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


def _naive_dft(x):
    n = x.shape[0]
    k = np.arange(n)
    return np.exp(-2j * np.pi * np.outer(k, k) / n) @ x


@pytest.mark.parametrize("n", [1, 2, 8, 64, 256, 1024])
def test_forward_matches_naive_dft(md, n):
    rng = np.random.default_rng(n)
    x = rng.normal(size=(n, 3)) + 1j * rng.normal(size=(n, 3))
    got = md.plan_fft(n).forward(x)
    want = _naive_dft(x)
    assert np.abs(got - want).max() <= 1e-10 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("n", [4, 512, 4096, 8192, 16384, 65536, 1 << 17, 1 << 20])
def test_forward_inverse_vs_oracle_and_round_trip(md, n):
    """Single-block lengths and the two-level lengths (> 4096) against the oracle's radix-2
    transform; inverse(forward(x)) = x."""
    from oracle.wr3l_oracle import plan as oplan
    rng = np.random.default_rng(7)
    x = rng.normal(size=(n, 2)) + 1j * rng.normal(size=(n, 2))
    p = md.plan_fft(n)
    f = p.forward(x)
    ref = oplan(n).forward(x)
    scale = np.abs(ref).max()
    assert np.abs(f - ref).max() <= 1e-12 * scale * np.log2(max(n, 2))
    back = p.inverse(f)
    assert np.abs(back - x).max() <= 1e-12 * np.log2(max(n, 2)) * np.abs(x).max()
    np.testing.assert_allclose(p.inverse(ref), oplan(n).inverse(ref), rtol=0, atol=1e-12 * np.abs(x).max() * 16)


def test_real_spectrum_api(md):
    rng = np.random.default_rng(3)
    s = rng.normal(size=256)
    p = md.plan_fft(256)
    sp = md.fft_forward_real(p, s)
    assert isinstance(sp, md.Spectrum) and sp.n == 256
    c = sp.coefficients
    np.testing.assert_allclose(c[1:], np.conj(c[1:][::-1]), rtol=0, atol=1e-11)    # Hermitian
    np.testing.assert_allclose(md.fft_inverse_real(p, sp), s, rtol=0, atol=1e-12)
    with pytest.raises(ValueError):
        md.fft_forward_real(p, np.zeros((4, 4)))
    with pytest.raises(ValueError):
        md.Spectrum(4, np.zeros(5))


def test_fft2_and_filters_vs_oracle(md):
    from oracle import wr3l_oracle as O
    rng = np.random.default_rng(11)
    g = md.Image(rng.uniform(0, 255, (64, 128)))
    spec = md.fft2_forward(g)
    np.testing.assert_allclose(spec, np.fft.fft2(g.values), rtol=0, atol=1e-9)
    back = md.fft2_inverse(spec)
    np.testing.assert_allclose(back.values, g.values, rtol=0, atol=1e-10)
    line = md.Psf.line(9.0, 30.0)
    op = O.OPsf("2d", line.weights, line.center)
    np.testing.assert_allclose(md.psf_spectrum_2d(line, (64, 128)), O.spectrum_2d(op, (64, 128)), rtol=0, atol=1e-12)
    box = md.Psf.uniform_box(md.BlurAxis.VERTICAL, 7.5)
    obox = O.make_psf("box", axis="v", length=7.5)
    p = md.plan_fft(64)
    h = md.psf_spectrum_1d(box, p)
    np.testing.assert_allclose(h, O.spectrum_1d(obox, 64), rtol=0, atol=1e-12)
    filt = O.wiener_multiplier(O.spectrum_1d(obox, 64), 0.006)
    a = rng.uniform(0, 255, (64, 7))                       # odd column count: the lone last column
    np.testing.assert_allclose(md.apply_column_filter(a, filt, p), O.column_filter(a, filt), rtol=0, atol=1e-9)
    q = rng.uniform(0, 1, (64, 7))
    pr, qr = md.filter_real_pair(a, q, filt, p)
    np.testing.assert_allclose(pr, O.column_filter(a, filt), rtol=0, atol=1e-9)
    np.testing.assert_allclose(qr, O.column_filter(q, filt), rtol=0, atol=1e-9)


def test_fft_api_errors(md):
    for n in (0, 3, 100, 1 << 21):                    # the reference's limit is 2^20 (fft.py:45)
        with pytest.raises(ValueError):
            md.FourierPlan(n)
    assert md.FourierPlan(1 << 20).n == 1 << 20
    with pytest.raises(ValueError):
        md.plan_fft(64).forward(np.zeros(32))


def test_device_tensors_stay_on_device(md):
    import torch
    x = torch.randn(128, 5, dtype=torch.complex128, device="cuda")
    y = md.plan_fft(128).forward(x)
    assert isinstance(y, torch.Tensor) and y.is_cuda
    np.testing.assert_allclose(y.cpu().numpy(), np.fft.fft(x.cpu().numpy(), axis=0), rtol=0, atol=1e-10)


@pytest.mark.parametrize("workers", [1, 3, 8])
def test_rrrl_deblur_parallel_equals_serial(md, workers):
    """Same result as rrrl_deblur with the same convolver, for any worker count (parallel.py)."""
    g = md.make_test_image(96, 64)                          # 64 rows: the vertical axis is a power of two
    for psf, conv in ((md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 9), "box"),
                      (md.Psf.general_1d([1, 3, 2, 1], md.BlurAxis.VERTICAL), "fourier")):
        f = md.synth_blur(g, psf)
        a = md.rrrl_deblur_parallel(f, psf, md.DeconvParams(), workers).values
        b = md.rrrl_deblur(f, psf, md.DeconvParams(), convolver=conv).values
        np.testing.assert_array_equal(a, b)
    with pytest.raises(ValueError):
        md.rrrl_deblur_parallel(g, md.Psf.line(5.0, 20.0), md.DeconvParams())
    with pytest.raises(ValueError):
        md.rrrl_deblur_parallel(g, md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 5), md.DeconvParams(), 0)


def test_array_level_convolutions_vs_oracle(md):
    """convolve_array / box_filter_array (conv.py:85-138) against the oracle's clamped direct
    summation and box filter, including a non-default box centre."""
    from oracle import wr3l_oracle as O
    rng = np.random.default_rng(5)
    a = rng.uniform(0, 255, (48, 64))
    line = md.Psf.line(7.0, 60.0)
    np.testing.assert_allclose(md.convolve_array(a, line), O.clamped_convolve(a, O.OPsf("2d", line.weights, line.center)),
                               rtol=0, atol=1e-9)
    for length, center, axis in ((9.0, 4, 0), (7.5, 2, 1), (12.0, 9, 0)):
        want = O.box_filter(a, length, center, axis=axis)
        np.testing.assert_allclose(md.box_filter_array(a, length, center, axis), want, rtol=0, atol=1e-9)


def test_column_sharpening_engine(md):
    """ColumnSharpeningEngine (parallel.py:43-114) through the step API equals rrrl_deblur."""
    from paper_1212_2245_b200.parallel import ColumnSharpeningEngine
    g = md.make_test_image(96, 64)
    psf = md.Psf.uniform_box(md.BlurAxis.VERTICAL, 9)
    f = md.synth_blur(g, psf)
    params = md.DeconvParams()
    fpos = np.maximum(f.values, params.floor)
    times = []
    eng = ColumnSharpeningEngine(params, None, 4)
    u = eng.run(fpos.copy(), fpos, md.make_convolver(psf, f.shape, "box"), params.iterations, times)
    want = md.rrrl_deblur(f, psf, params, convolver="box").values
    np.testing.assert_allclose(u, want, rtol=0, atol=1e-9)
    assert len(times) == params.iterations
    with pytest.raises(ValueError):
        ColumnSharpeningEngine(params, None, 0)


def test_rrrl_deblur_parallel_with_object_convolver(md):
    """A convolver OBJECT passed to rrrl_deblur_parallel sees the frame in vertical orientation
    (horizontal kernels transposed around the call, parallel.py:130-142), as in the reference."""
    from oracle import wr3l_oracle as O
    g = md.make_test_image(64, 48)
    psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 9)
    f = md.synth_blur(g, psf)
    obj = O.BoxConv(9.0, 4, 9, axis=0)                  # acts along axis 0 of what it is given
    got = md.rrrl_deblur_parallel(f, psf, md.DeconvParams(), 3, convolver=obj).values
    want = md.rrrl_deblur(f, psf, md.DeconvParams(), convolver="box").values
    assert np.abs(got - want).max() <= 1e-8
