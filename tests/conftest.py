"""Shared fixtures. ``gpu``-marked tests need a B200 (run via gpurun); all others run on CPU."""

from __future__ import annotations

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden_names(prefix: str = "") -> list[str]:
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        d = {k: z[k] for k in z.files}
    for k in ("f", "g"):
        if k in d:
            d[k] = d[k].astype(np.float64)
    return d


def oracle_psf(d: dict):
    """OPsf from a fixture's psf_* fields (weights are stored already normalised)."""
    from oracle.wr3l_oracle import OPsf
    kind = str(d["psf_kind"])
    c = d["psf_center"]
    axis = str(d["psf_axis"]) or None
    length = float(d["psf_length"])
    center = (int(c[0]), int(c[1])) if kind == "2d" else int(c[0])
    return OPsf(kind, d["psf_weights"], center, axis, None if np.isnan(length) else length)


def oracle_params(d: dict):
    from oracle.wr3l_oracle import OParams
    k, a, it, ed, er, fl = (float(v) for v in d["params"])
    return OParams(k, a, int(it), ed, er, fl)


def product_psf(d: dict):
    """Product ``Psf`` with exactly the fixture's (normalised) weights."""
    from paper_1212_2245_b200.core import BlurAxis, Psf, PsfKind
    kind = PsfKind(str(d["psf_kind"]))
    c = d["psf_center"]
    axis = str(d["psf_axis"])
    length = float(d["psf_length"])
    w = np.array(d["psf_weights"], dtype=np.float64)
    w.setflags(write=False)
    if kind is PsfKind.GENERAL_2D:
        return Psf(kind, w, (int(c[0]), int(c[1])))
    return Psf(kind, w, int(c[0]), axis=BlurAxis(axis), length=None if np.isnan(length) else length)


def product_params(d: dict):
    from paper_1212_2245_b200.core import DeconvParams
    k, a, it, ed, er, fl = (float(v) for v in d["params"])
    return DeconvParams(k, a, int(it), ed, er, fl)


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
