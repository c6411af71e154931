"""PGM I/O and CLI plumbing on CPU (the reference's test_pgm.py / test_cli.py for the kept parts)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1212_2245_b200 as md
from paper_1212_2245_b200.cli import main, parse_psf_spec, UsageError


def test_pgm_round_trip(tmp_path):
    img = md.make_test_image(40, 30)
    p = tmp_path / "a.pgm"
    md.write_pgm(img, p)
    back = md.read_pgm(p)
    np.testing.assert_array_equal(back.values, img.values)
    assert back.shape == (30, 40)


def test_pgm_rounds_half_up_and_clamps(tmp_path):
    p = tmp_path / "b.pgm"
    md.write_pgm(md.Image([[-3.0, 2.5, 254.5, 300.0]]), p)
    np.testing.assert_array_equal(md.read_pgm(p).values, [[0.0, 3.0, 255.0, 255.0]])


def test_pgm_comments_and_errors(tmp_path):
    p = tmp_path / "c.pgm"
    p.write_bytes(b"P5\n# comment\n2 1\n255\n\x01\x02")
    np.testing.assert_array_equal(md.read_pgm(p).values, [[1.0, 2.0]])
    p.write_bytes(b"P2\n2 1\n255\n12")
    with pytest.raises(ValueError):
        md.read_pgm(p)
    p.write_bytes(b"P5\n4 4\n255\n\x00")
    with pytest.raises(ValueError):
        md.read_pgm(p)


def test_psf_specs():
    assert parse_psf_spec("box:h:15").length == 15.0
    assert parse_psf_spec("line:21:30").weights.shape == (25, 25)
    with pytest.raises(UsageError):
        parse_psf_spec("disc:3")


def test_cli_usage_errors(tmp_path):
    assert main(["testimage", str(tmp_path / "t.pgm"), "--width", "32", "--height", "16"]) == 0
    assert md.read_pgm(tmp_path / "t.pgm").shape == (16, 32)
    assert main(["deblur", str(tmp_path / "t.pgm"), str(tmp_path / "o.pgm"), "--psf", "nope"]) == 1
    assert main(["nosuchcommand"]) == 1
    assert main(["deblur", str(tmp_path / "missing.pgm"), str(tmp_path / "o.pgm"), "--psf", "box:h:3"]) == 2


def test_deblur_parser_accepts_reference_threads_flag():
    from paper_1212_2245_b200.cli import build_parser
    a = build_parser().parse_args(["deblur", "in.pgm", "out.pgm", "--psf", "box:h:15", "--threads", "8"])
    assert a.threads == 8
