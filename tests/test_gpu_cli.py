"""CLI deblur / bench on the GPU through the public API."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def md():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1212_2245_b200 as m
    return m


def test_cli_deblur_matches_api(md, tmp_path, capsys):
    from paper_1212_2245_b200.cli import main
    psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 9)
    f = md.synth_blur(md.make_test_image(64, 64), psf)
    md.write_pgm(f, tmp_path / "f.pgm")
    assert main(["deblur", str(tmp_path / "f.pgm"), str(tmp_path / "u.pgm"), "--psf", "box:h:9", "--time"]) == 0
    out = capsys.readouterr().out
    assert "wiener:" in out and "total:" in out
    want = md.wr3l(f, psf, md.DeconvParams())
    got = md.read_pgm(tmp_path / "u.pgm").values
    np.testing.assert_array_equal(got, np.clip(np.floor(want.values + 0.5), 0, 255))
    # and against the CPU oracle of the reference's `motiondeblur deblur` (cli.py:132-167: wr3l,
    # then write_pgm's round-half-up quantisation); a pixel may differ by one grey level only
    # where the unquantised values straddle a .5 boundary within the parity bar
    from oracle import wr3l_oracle as O
    ref = O.pipeline(f.values, O.make_psf("box", axis="h", length=9), O.OParams(), "box")
    ref_q = np.clip(np.floor(ref + 0.5), 0, 255)
    diff = np.abs(got - ref_q)
    assert diff.max() <= 1.0
    near = np.abs((ref + 0.5) - np.round(ref + 0.5)) <= 1e-4 * 255
    assert np.all((diff == 0) | near)


def test_cli_deblur_threads_flag(md, tmp_path):
    """The reference's --threads (cli.py:215) is accepted; the output does not depend on it."""
    from paper_1212_2245_b200.cli import main
    psf = md.Psf.uniform_box(md.BlurAxis.VERTICAL, 7)
    md.write_pgm(md.synth_blur(md.make_test_image(64, 32), psf), tmp_path / "f.pgm")
    assert main(["deblur", str(tmp_path / "f.pgm"), str(tmp_path / "a.pgm"), "--psf", "box:v:7"]) == 0
    assert main(["deblur", str(tmp_path / "f.pgm"), str(tmp_path / "b.pgm"), "--psf", "box:v:7", "--threads", "4"]) == 0
    np.testing.assert_array_equal(md.read_pgm(tmp_path / "a.pgm").values, md.read_pgm(tmp_path / "b.pgm").values)


def test_cli_bench_csv(md, tmp_path, capsys):
    from paper_1212_2245_b200.cli import main
    md.write_pgm(md.make_test_image(64, 64), tmp_path / "f.pgm")
    assert main(["bench", str(tmp_path / "f.pgm"), "--psf", "box:v:7", "--runs", "3", "--format", "csv"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "scenario,stage,runs,mean_ms,std_ms,min_ms,max_ms"
    assert {l.split(",")[1] for l in lines[1:]} == {"wiener", "rrrl_iteration", "rrrl_total", "total"}


def test_lut_r1_on_device(md):
    lut = md.default_divergence_lut()
    xs = np.array([0.03125, 0.2, 0.5, 1.0, 3.7, 64.9, 65.0, 100.0])
    got = lut.r1(xs)
    assert got[3] == 0.0
    direct = xs - 1 - np.log(xs)
    assert np.abs(got[:-1] - direct[:-1]).max() < 1e-4
    # above the table: linear continuation matching value and slope at 65 (deconv.py:127-129)
    assert got[-1] == pytest.approx(65.0 - 1 - np.log(65.0) + (1 - 1 / 65) * 35.0, abs=1e-12)
    assert lut.table.shape == (133057,)
