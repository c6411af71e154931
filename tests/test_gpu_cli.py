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
