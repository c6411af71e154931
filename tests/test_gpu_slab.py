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
