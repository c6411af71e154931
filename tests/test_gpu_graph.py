"""CUDA-graph capture of the pipeline (GpuPlan.capture / DeblurPipeline.capture, md_run under
stream capture): replays equal direct runs bit for bit on the line path (fused cluster kernel
and per-iteration kernels, chunked), the 2D path and float64; new frames written into the input
buffer are picked up; a capture that would need more scratch than the warm-up sized fails."""

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


def _frames(md, shape, psf, n, seed):
    return np.stack([md.synth_blur(md.make_test_image(shape[1], shape[0], seed=seed + i), psf).values
                     for i in range(n)])


@pytest.mark.parametrize("case", ["box_f32_fused", "box_f32_chunked", "box_f64", "line_2d_f32"])
def test_replay_equals_run(md, case):
    import torch
    if case.startswith("box"):
        psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15.0)
        shape, scen = (64, 128), md.Scenario.BOX_1D
    else:
        psf = md.Psf.line(9.0, 30.0)
        shape, scen = (64, 64), md.Scenario.FOURIER_2D
    dtype = "float64" if case.endswith("f64") else "float32"
    pipe = md.DeblurPipeline(shape, psf, md.DeconvParams(), scen, dtype=dtype)
    n = 6
    if case.endswith("chunked"):
        pipe.plan.set_fused(False)
        pipe.plan.set_chunk(2)
    g = pipe.capture(n)
    for seed in (0, 40):                                  # two batches through one graph
        x = torch.from_numpy(_frames(md, shape, psf, n, seed)).to("cuda", g.f.dtype)
        got = g(x).clone()
        want = pipe.run_batch(x)
        torch.cuda.synchronize()
        assert torch.equal(got, want), case


def test_replay_on_side_stream(md):
    import torch
    psf = md.Psf.uniform_box(md.BlurAxis.VERTICAL, 9.0)
    pipe = md.DeblurPipeline((128, 32), psf, md.DeconvParams(), dtype="float32")
    g = pipe.capture(3)
    x = torch.from_numpy(_frames(md, (128, 32), psf, 3, 7)).to("cuda", torch.float32)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    out = g(x, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    assert torch.equal(out, pipe.run_batch(x))


def test_capture_cannot_grow_scratch(md):
    """The plan's scratch is sized by the warm-up run; a capture of a larger batch on the same
    plan would reallocate it under a live graph and is refused."""
    import torch
    psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 7.0)
    plan = md.DeblurPipeline((32, 64), psf, md.DeconvParams(), dtype="float32", fused=False).plan
    plan.set_chunk(1 << 20)
    f = torch.full((2, 32, 64), 10.0, device="cuda")
    plan.capture(f)                                       # sizes scratch for 2 frames
    big = torch.full((64, 32, 64), 10.0, device="cuda")
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    with pytest.raises((ValueError, RuntimeError)):
        with torch.cuda.graph(graph, stream=side, capture_error_mode="relaxed"):
            plan.run(big, stream=side)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(plan.run(f).cpu().numpy(), plan.run(f).cpu().numpy())


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_graph_survives_scratch_growth(md, dtype):
    """A graph captured for one frame stays valid after an uncaptured run of a larger batch grew
    the plan's scratch (the captured buffer is retired, not freed): replay still equals run."""
    import torch
    psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15.0)
    pipe = md.DeblurPipeline((64, 128), psf, md.DeconvParams(), md.Scenario.BOX_1D, dtype=dtype)
    g = pipe.capture(1)
    tdt = torch.float32 if dtype == "float32" else torch.float64
    big = torch.from_numpy(_frames(md, (64, 128), psf, 64, 3)).to("cuda", tdt)
    pipe.run_batch(big)                                   # grows the scratch
    junk = torch.full((1 << 22,), 7.0, device="cuda")     # reuse of freed memory would show here
    x = torch.from_numpy(_frames(md, (64, 128), psf, 1, 90)).to("cuda", tdt)
    got = g(x).clone()
    want = pipe.run_batch(x)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    del junk
