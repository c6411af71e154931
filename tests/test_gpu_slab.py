"""Row-slab decomposition of one image (BASELINE.json configs[4]) on the GPU.

The slab driver (paper_1212_2245_b200/slab.py) runs its SPMD program with one thread per
"rank" inside this process (LocalComm: host barriers + device copies; no kernel waits on
another), so the per-slab CUDA kernels, the halo geometry, the periodic wrap and the two
spectrum transposes are exercised exactly as on 8 GPUs. The result must equal the
single-plan run of the same image.
"""

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


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_slabs_equal_single_plan(md, world):
    import torch
    from paper_1212_2245_b200.slab import run_slabs
    n = 512
    psf = md.Psf.line(21.0, 30.0)
    f = torch.from_numpy(md.synth_blur(md.make_test_image(n, n), psf).values.copy()).cuda()
    pipe = md.DeblurPipeline((n, n), psf, md.DeconvParams(iterations=3), big_fft=True)
    want = pipe.run_batch(f)
    got = run_slabs(pipe.plan, f, world)
    assert float((got - want).abs().max()) <= 1e-9


def test_slabs_match_oracle(md):
    from oracle import wr3l_oracle as O
    import torch
    from paper_1212_2245_b200.slab import run_slabs
    n = 256
    psf = md.Psf.line(15.0, 120.0)
    g = md.make_test_image(n, n)
    f = md.synth_blur(g, psf)
    pipe = md.DeblurPipeline((n, n), psf, md.DeconvParams(), big_fft=True)
    got = run_slabs(pipe.plan, torch.from_numpy(f.values.copy()).cuda(), 4).cpu().numpy()
    ref = O.pipeline(f.values, O.OPsf("2d", psf.weights, psf.center), O.OParams(), "fourier2d")
    assert np.abs(got - ref).max() <= 1e-6


def test_slab_plan_requirements(md):
    from paper_1212_2245_b200.slab import CudaSlabBackend
    pipe = md.DeblurPipeline((64, 64), md.Psf.line(9.0, 10.0), md.DeconvParams())     # no big_fft
    with pytest.raises(ValueError):
        CudaSlabBackend(pipe.plan)


def _c5_golden():
    import os
    from conftest import GOLDEN
    path = os.path.join(GOLDEN, "big_c5_4096.npz")
    if not os.path.exists(path):
        pytest.skip("big_c5_4096.npz not generated")
    return np.load(path)


def _check_against_c5_golden(md, d, u, g):
    """Size-independent comparison with the reference's 4096^2 c5 run (oracle/gen_golden_c5.py):
    the slab-boundary rows, 20,000 seeded pixels, row / column means, PSNR."""
    tol = 1e-4 * 255.0
    rows = d["rows"]
    assert float(np.abs(u[rows] - d["row_values"]).max()) <= tol
    assert float(np.abs(u[d["py"], d["px"]] - d["pix_values"]).max()) <= tol
    assert float(np.abs(u.mean(axis=1) - d["row_means"]).max()) <= tol
    assert float(np.abs(u.mean(axis=0) - d["col_means"]).max()) <= tol
    psnr = 10.0 * np.log10(255.0 ** 2 / np.mean((u - g) ** 2))
    assert abs(psnr - float(d["psnr"])) <= 0.01


@pytest.fixture(scope="module")
def c5_input(md):
    """The reference's c5 input at 4096^2, regenerated here (scene + GPU synth blur) and checked
    byte for byte against the fixture's hash."""
    import hashlib
    import torch
    d = _c5_golden()
    psf = md.Psf.general_2d(d["psf_weights"], center=tuple(int(c) for c in d["psf_center"]))
    g = md.make_test_image(4096, 4096, seed=7).values
    f = md.synth_blur(md.Image(g), psf).values
    assert hashlib.sha256(np.ascontiguousarray(f).tobytes()).hexdigest() == str(d["f_sha256"])
    return d, psf, g, torch.from_numpy(f.copy()).cuda()


def test_c5_4096_single_plan_vs_reference(md, c5_input):
    """c5 pinned at 4096^2 against the reference's own FOURIER_2D run: the
    two-level-FFT Wiener plus direct-tap iterations of one plan (big_fft, as the c5 bench runs)."""
    d, psf, g, f = c5_input
    pipe = md.DeblurPipeline((4096, 4096), psf, md.DeconvParams(), md.Scenario.FOURIER_2D, big_fft=True)
    u = pipe.run_batch(f).cpu().numpy()
    _check_against_c5_golden(md, d, u, g)


def test_c5_4096_eight_slabs_vs_reference(md, c5_input):
    """The same image as 8 row slabs (the 8-GPU split of configs[4], thread ranks here)."""
    from paper_1212_2245_b200.slab import run_slabs
    d, psf, g, f = c5_input
    pipe = md.DeblurPipeline((4096, 4096), psf, md.DeconvParams(), md.Scenario.FOURIER_2D, big_fft=True)
    u = run_slabs(pipe.plan, f, 8).cpu().numpy()
    _check_against_c5_golden(md, d, u, g)


def test_c5_16384_eight_slabs_equal_single_plan(md):
    """configs[4] at its real size: 16384^2, line L=21 @30 deg, 5 iterations -- 8 row slabs
    against the single plan (1e-9), plus sanity of the result (finite, positive, mean kept).
    The reference itself is pinned on this path at 4096^2 (the tests above)."""
    import torch
    from paper_1212_2245_b200.slab import run_slabs
    n = 16384
    psf = md.Psf.line(21.0, 30.0)
    yy = torch.linspace(0, 1, n, device="cuda", dtype=torch.float64)
    gen = torch.Generator(device="cuda").manual_seed(5)
    blocks = torch.rand((n // 64, n // 64), generator=gen, device="cuda", dtype=torch.float64)
    g = 60.0 + 100.0 * yy[:, None] + 60.0 * yy[None, :]
    g = g + 40.0 * (blocks.repeat_interleave(64, 0).repeat_interleave(64, 1) - 0.5)
    conv = md.make_convolver(psf, (n, n), "spatial")
    f = torch.clamp(torch.floor(conv.blur(g.contiguous()) + 0.5), 0, 255)
    del blocks
    pipe = md.DeblurPipeline((n, n), psf, md.DeconvParams(), big_fft=True)
    want = pipe.run_batch(f)
    got = run_slabs(pipe.plan, f, 8)
    assert float((got - want).abs().max()) <= 1e-9
    assert bool(torch.isfinite(want).all())
    assert float(want.min()) > 0.0                     # the multiplicative update keeps u positive
    assert abs(float(want.mean()) - float(f.mean())) < 1.0   # RL-type updates preserve the mean


def test_slab_bands_enable_overlap(md):
    """The band split the worker uses to overlap the halo exchange with the interior rows
    (md_slab_bands / md_slab_stage): margins cover the blur and adjoint halos, and the c5 slabs
    (2048 rows at 8 ranks) are deep enough for it."""
    from paper_1212_2245_b200.slab import CudaSlabBackend
    pipe = md.DeblurPipeline((512, 512), md.Psf.line(21.0, 30.0), md.DeconvParams(), big_fft=True)
    be = CudaSlabBackend(pipe.plan)
    a_in, b_in = be.bands()
    top, bot = be.halo_rows()
    ht, hb = be.adj_halo
    assert a_in >= 1 and b_in >= a_in + max(ht, hb) and b_in >= 2
    assert top >= ht + a_in - 1 and bot >= hb + a_in - 1
    assert 2 * b_in <= 16384 // 8
