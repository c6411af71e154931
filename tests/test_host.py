"""Host-side data model and input tooling (no GPU): mirrors test_core.py / test_synth.py of
the reference for the pieces the drop-in keeps."""

from __future__ import annotations

import math
import warnings

import numpy as np
import pytest

import paper_1212_2245_b200 as md
from conftest import load_golden
from paper_1212_2245_b200.core import BlurAxis, Psf, PsfKind


class TestBoxKernel:
    def test_integer_length(self):
        np.testing.assert_array_equal(md.materialize_box_kernel(5), np.full(5, 0.2))

    def test_fractional_length(self):
        w = md.materialize_box_kernel(21.5)
        assert w.shape == (23,)
        assert w[0] == w[-1] == pytest.approx(0.5 / 43.0)
        assert w.sum() == pytest.approx(1.0, abs=1e-12)

    @pytest.mark.parametrize("bad", [0.5, 0.0, -3, float("nan"), float("inf")])
    def test_rejects(self, bad):
        with pytest.raises(ValueError):
            md.materialize_box_kernel(bad)


class TestPsf:
    def test_general_2d_normalises_and_centres(self):
        p = Psf.general_2d(np.ones((3, 5)))
        assert p.center == (1, 2)
        assert p.weights.sum() == pytest.approx(1.0)
        assert not p.weights.flags.writeable

    def test_general_1d_center_default(self):
        p = Psf.general_1d([1, 2, 3, 4], BlurAxis.HORIZONTAL)
        assert p.center == 2 and p.support == (1, 4)

    def test_uniform_box(self):
        p = Psf.uniform_box(BlurAxis.VERTICAL, 15)
        assert p.kind is PsfKind.UNIFORM_BOX_1D and p.center == 7 and p.length == 15.0
        assert p.support == (15, 1)

    @pytest.mark.parametrize("w", [[], [-1.0, 2.0], [0.0, 0.0], [np.nan]])
    def test_rejects_bad_weights(self, w):
        with pytest.raises(ValueError):
            Psf.general_1d(w, BlurAxis.VERTICAL)

    def test_rejects_center_outside(self):
        with pytest.raises(ValueError):
            Psf.general_2d(np.ones((3, 3)), center=(3, 0))
        with pytest.raises(ValueError):
            Psf.general_1d([1, 1], BlurAxis.VERTICAL, center=2)

    def test_adjoint_involution(self, rng):
        p = Psf.general_2d(rng.uniform(0, 1, (4, 5)), center=(1, 3))
        q = md.adjoint(md.adjoint(p))
        np.testing.assert_array_equal(q.weights, p.weights)
        assert q.center == p.center
        a = md.adjoint(p)
        assert a.center == (2, 1)
        np.testing.assert_array_equal(a.weights, p.weights[::-1, ::-1])

    def test_line_psf(self):
        p = Psf.line(21.0, 30.0)
        assert p.kind is PsfKind.GENERAL_2D and p.weights.shape == (25, 25) and p.center == (12, 12)
        assert p.weights.sum() == pytest.approx(1.0, abs=1e-12)
        ys, xs = np.mgrid[0:25, 0:25]
        cx = float((p.weights * xs).sum()) - 12
        cy = float((p.weights * ys).sum()) - 12
        assert abs(cx) < 1e-9 and abs(cy) < 1e-9            # centred segment
        nnz = int((p.weights > 0).sum())
        assert 40 <= nnz <= 90
        h = Psf.line(9.0, 0.0)
        assert np.count_nonzero(h.weights.sum(axis=1)) == 1   # horizontal: one row

    def test_line_psf_deterministic(self):
        np.testing.assert_array_equal(Psf.line(17.5, 42.0).weights, Psf.line(17.5, 42.0).weights)


class TestParams:
    def test_defaults(self):
        p = md.DeconvParams()
        assert (p.wiener_k, p.alpha, p.iterations, p.eps_data, p.eps_reg, p.floor) == (
            0.006, 0.003, 5, 1.0, 0.01, 0.1)

    @pytest.mark.parametrize("kw", [dict(wiener_k=0), dict(alpha=-1), dict(iterations=-1),
                                    dict(iterations=2.5), dict(eps_data=0), dict(eps_reg=0), dict(floor=0)])
    def test_validation(self, kw):
        with pytest.raises(ValueError):
            md.DeconvParams(**kw)


class TestParsePsf:
    def test_box(self):
        p = md.parse_psf("BOX h 9.5")
        assert p.kind is PsfKind.UNIFORM_BOX_1D and p.axis is BlurAxis.HORIZONTAL and p.length == 9.5

    def test_1d_and_2d(self):
        p = md.parse_psf("1D v 3 0\n0.25 0.5 0.25")
        assert p.center == 0 and p.axis is BlurAxis.VERTICAL
        q = md.parse_psf("2D 3 2 2 1\n1 1 1\n1 1 1")
        assert q.weights.shape == (2, 3) and q.center == (1, 2)

    def test_warns_on_renormalisation(self):
        with pytest.warns(UserWarning):
            md.parse_psf("1D v 2 0 3 3")
        with warnings.catch_warnings():
            warnings.simplefilter("error")
            md.parse_psf("1D v 2 0 0.5 0.5")

    @pytest.mark.parametrize("txt", ["", "BOX h", "1D v 3 0 1 2", "2D 2 2 0 0 1", "XD 1"])
    def test_rejects(self, txt):
        with pytest.raises(ValueError):
            md.parse_psf(txt)


class TestImage:
    def test_copy_and_readonly(self):
        a = np.ones((3, 4))
        img = md.Image(a)
        a[0, 0] = 5
        assert img.values[0, 0] == 1 and not img.values.flags.writeable
        assert img.shape == (3, 4) and img.height == 3 and img.width == 4

    @pytest.mark.parametrize("bad", [np.ones(3), np.ones((0, 3)), np.array([[np.inf]])])
    def test_rejects(self, bad):
        with pytest.raises(ValueError):
            md.Image(bad)

    def test_clamp_floor(self):
        out = md.clamp_floor(md.Image([[-1.0, 0.05, 3.0]]), 0.1)
        np.testing.assert_array_equal(out.values, [[0.1, 0.1, 3.0]])
        with pytest.raises(ValueError):
            md.clamp_floor(md.Image([[1.0]]), 0.0)


class TestSynth:
    def test_scene_matches_reference_fixture(self):
        d = load_golden("pipe_c1_box_h15_256")
        np.testing.assert_array_equal(md.make_test_image(256, 256, seed=7).values, d["g"])

    def test_scene_non_square(self):
        d = load_golden("pipe_box_v21p5_64x96")
        assert md.make_test_image(96, 64).shape == (64, 96)
        np.testing.assert_array_equal(md.make_test_image(96, 64).values, d["g"])

    def test_noise_is_pcg64(self):
        img = md.Image(np.full((8, 8), 100.0))
        a = md.add_gaussian_noise(img, 5.0, seed=5).values
        b = np.clip(100.0 + np.random.default_rng(5).normal(0.0, 5.0, (8, 8)), 0, 255)
        np.testing.assert_array_equal(a, b)

    def test_quantize(self):
        np.testing.assert_array_equal(md.quantize(md.Image([[-3.0, 2.5, 254.6, 300.0]])).values,
                                      [[0.0, 3.0, 255.0, 255.0]])

    def test_snr_and_psnr(self):
        g = md.make_test_image(32, 32)
        assert md.snr(g, g) == math.inf
        assert md.psnr(g.values, g.values) == math.inf
        assert md.psnr(g.values + 1.0, g.values) == pytest.approx(10 * math.log10(255.0 ** 2))


class TestPsfBankGrouping:
    def test_groups_of_sorted_index(self):
        from paper_1212_2245_b200.batch import PsfBankPipeline
        g = PsfBankPipeline.groups(None, np.array([0, 0, 1, 3, 3, 3]))
        assert g == [(0, 0, 2), (1, 2, 3), (3, 3, 6)]
        assert PsfBankPipeline.groups(None, np.array([], dtype=np.int64)) == []
        with pytest.raises(ValueError):
            PsfBankPipeline.groups(None, np.array([1, 0]))


def test_fft_api_host_side():
    """Host-side pieces of the transform API (paper_1212_2245_b200/fft.py): PSF embedding equals
    the oracle's (fft.py:192-221), plan validation as the reference (fft.py:62-66), and no CPU
    fallback for the transform itself."""
    import paper_1212_2245_b200 as md
    from oracle import wr3l_oracle as O
    box = md.Psf.uniform_box(md.BlurAxis.VERTICAL, 7.5)
    np.testing.assert_array_equal(md.embed_psf_1d(box, 32), O.embed_1d(O.make_psf("box", axis="v", length=7.5), 32))
    line = md.Psf.line(9.0, 30.0)
    np.testing.assert_array_equal(md.embed_psf_2d(line, (32, 64)), O.embed_2d(O.OPsf("2d", line.weights, line.center), (32, 64)))
    for n in (0, 3, 1 << 21):                # the reference allows up to 2^20 (fft.py:45)
        with pytest.raises(ValueError):
            md.FourierPlan(n)
    with pytest.raises(ValueError):
        md.embed_psf_1d(md.Psf.uniform_box(md.BlurAxis.VERTICAL, 31), 16)
    import torch
    if not torch.cuda.is_available():
        with pytest.raises((md._lib.CudaUnavailable, RuntimeError)):
            md.plan_fft(8).forward(np.ones(8))


def test_benchmark_report_formats_match_reference():
    """report() renders the reference's human table and CSV byte for byte (bench.py:118-138);
    the expected strings were produced by the reference's own report() on these samples."""
    from paper_1212_2245_b200.benchmark import StageStats, TimingStats, report
    st = {k: StageStats.from_samples(v) for k, v in {"wiener": [1.0, 1.5, 2.0], "rrrl_iteration": [0.25, 0.5, 0.75, 1.25],
          "rrrl_total": [3.0], "total": [4.0, 4.5]}.items()}
    ts = TimingStats("box", 3, st)
    assert report(ts, "human") == (
        "scenario box, 3 runs\n  wiener             1.500 +-  0.500 ms  (1.000 .. 2.000, n=3)\n"
        "  rrrl_iteration     0.688 +-  0.427 ms  (0.250 .. 1.250, n=4)\n"
        "  rrrl_total         3.000 +-  0.000 ms  (3.000 .. 3.000, n=1)\n"
        "  total              4.250 +-  0.354 ms  (4.000 .. 4.500, n=2)\n")
    assert report(ts, "csv") == (
        "scenario,stage,runs,mean_ms,std_ms,min_ms,max_ms\nbox,wiener,3,1.500,0.500,1.000,2.000\n"
        "box,rrrl_iteration,4,0.688,0.427,0.250,1.250\nbox,rrrl_total,1,3.000,0.000,3.000,3.000\n"
        "box,total,2,4.250,0.354,4.000,4.500\n")
    assert StageStats.from_samples([]) == StageStats(0, 0.0, 0.0, 0.0, 0.0)
    assert StageStats.from_samples([2.0]) == StageStats(1, 2.0, 0.0, 2.0, 2.0)
    assert ts.mean_ms == st["total"].mean_ms and ts.max_ms == 4.5
    with pytest.raises(ValueError):
        report(ts, "xml")


@pytest.mark.parametrize("kw, expect", [
    (dict(wiener_k=0, iterations=float("inf")), ("ValueError", "wiener_k must be positive")),
    (dict(wiener_k=0, eps_data=None), ("ValueError", "wiener_k must be positive")),
    (dict(iterations=float("nan")), ("ValueError", "cannot convert float NaN to integer")),
    (dict(iterations=float("inf")), ("OverflowError", "cannot convert float infinity to integer")),
    (dict(iterations=2.5), ("ValueError", "iterations must be a non-negative integer")),
    (dict(alpha=-1), ("ValueError", "alpha must be non-negative")),
    (dict(alpha=float("nan")), None),
    (dict(floor=0), ("ValueError", "eps_data, eps_reg and floor must be positive")),
    (dict(eps_reg=float("nan")), ("ValueError", "eps_data, eps_reg and floor must be positive")),
    (dict(eps_data=None), ("TypeError", None)),
])
def test_deconv_params_checks_short_circuit_like_reference(kw, expect):
    """Outcomes recorded from the reference's DeconvParams (core.py:249-257): the first failing
    check raises, with the reference's comparison forms (NaN / inf / None behave the same)."""
    import paper_1212_2245_b200 as md
    if expect is None:
        md.DeconvParams(**kw)
        return
    with pytest.raises(Exception) as ei:
        md.DeconvParams(**kw)
    assert type(ei.value).__name__ == expect[0]
    if expect[1]:
        assert str(ei.value) == expect[1]


def test_fft_module_exports_fourier_convolve():
    from paper_1212_2245_b200 import fft
    assert "fourier_convolve" in fft.__all__ and callable(fft.fourier_convolve)


def test_rl_deblur_iterations_are_a_range_bound():
    """rl_deblur's iteration count is a range() bound as in the reference (deconv.py:531):
    a fractional count raises TypeError before any device work."""
    import paper_1212_2245_b200 as md
    f = md.Image(np.full((8, 8), 10.0))
    with pytest.raises(TypeError):
        md.rl_deblur(f, md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 3), 2.5)
