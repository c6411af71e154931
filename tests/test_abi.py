"""The C-ABI library loads and exports every symbol include/mdcuda.h declares; the ctypes
mirror of md_plan_desc matches the C layout. CPU-only (no compute calls)."""

from __future__ import annotations

import ctypes
import os
import re
import shutil
import subprocess

import pytest

from conftest import ROOT
from paper_1212_2245_b200 import _lib

HEADER = os.path.join(ROOT, "include", "mdcuda.h")


def declared_functions() -> list[str]:
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(md_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("md_plan_create", "md_run", "md_run_host", "md_wiener", "md_convolve",
                 "md_adjoint_pair", "md_rrrl_step", "md_robust_weight", "md_diffusion"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_signatures_cover_header():
    assert set(declared_functions()) == set(_lib.SIGNATURES)


def test_abi_version():
    assert _lib.load_library().md_abi_version() == 1


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")
def test_plan_desc_layout_matches_c(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "mdcuda.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu\\n\", sizeof(md_plan_desc),"
        " offsetof(md_plan_desc, box_length), offsetof(md_plan_desc, psf_weights),"
        " offsetof(md_plan_desc, flags), offsetof(md_plan_desc, floor)); return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    D = _lib.PlanDesc
    want = [ctypes.sizeof(D), D.box_length.offset, D.psf_weights.offset, D.flags.offset, D.floor.offset]
    assert got == want


def test_error_path_without_device_is_loud():
    """No CPU fallback: without a CUDA device every compute entry raises."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1212_2245_b200 as md
    f = md.Image(__import__("numpy").ones((16, 16)))
    with pytest.raises(_lib.CudaUnavailable):
        md.wr3l(f, md.Psf.uniform_box(md.BlurAxis.VERTICAL, 3), md.DeconvParams())
