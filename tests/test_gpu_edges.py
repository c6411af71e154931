"""Edge cases of the CUDA path against the CPU oracle: empty and ragged
batches, extreme observations (all zero, saturated, impulse noise), the longest supported blur
axis and the limits just past it. Oracle-checked at sizes the NumPy restatement finishes in
seconds; bar max|d| <= 1e-4 * 255 (north_star)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4 * 255.0


@pytest.fixture(scope="module")
def md():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1212_2245_b200 as md
    return md


def _oracle(md, f, psf, params, scenario):
    from oracle import wr3l_oracle as O
    if psf.kind.value == "box":
        op = O.make_psf("box", axis="h" if psf.axis == md.BlurAxis.HORIZONTAL else "v", length=psf.length)
    elif psf.kind.value == "1d":
        op = O.make_psf("1d", weights=psf.weights, center=psf.center,
                        axis="h" if psf.axis == md.BlurAxis.HORIZONTAL else "v")
    else:
        op = O.OPsf("2d", psf.weights, psf.center)
    p = O.OParams(wiener_k=params.wiener_k, alpha=params.alpha, iterations=params.iterations,
                  eps_data=params.eps_data, eps_reg=params.eps_reg, floor=params.floor)
    return O.pipeline(np.asarray(f, dtype=np.float64), op, p, scenario)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_empty_batch(md, dtype):
    import torch
    pipe = md.DeblurPipeline((64, 64), md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 7), md.DeconvParams(), dtype=dtype)
    tdt = torch.float64 if dtype == "float64" else torch.float32
    out = pipe.run_batch(torch.empty((0, 64, 64), device="cuda", dtype=tdt))
    assert tuple(out.shape) == (0, 64, 64)
    host = pipe.run_batch(np.empty((0, 64, 64), dtype=np.uint8), out_dtype=np.float32)
    assert host.shape == (0, 64, 64)


@pytest.mark.parametrize("n", [1, 3, 33, 35])
def test_ragged_batch_sizes_fused(md, n):
    """Batch sizes around the resident-cluster count of the fused kernel: each frame as alone."""
    import torch
    psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15)
    pipe = md.DeblurPipeline((256, 256), psf, md.DeconvParams(), dtype="float32")
    assert pipe.plan.fused
    g = md.make_test_image(256, 256)
    base = md.quantize(md.add_gaussian_noise(md.synth_blur(g, psf), 5.0, seed=1)).values
    frames = np.stack([np.roll(base, 7 * i, axis=0) for i in range(n)])
    out = pipe.run_batch(torch.from_numpy(frames).cuda().float()).cpu().numpy()
    for i in (0, n - 1):
        one = pipe.run_batch(torch.from_numpy(frames[i:i + 1]).cuda().float()).cpu().numpy()[0]
        np.testing.assert_array_equal(out[i], one)


@pytest.mark.parametrize("kind", ["zeros", "saturated", "impulse"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_extreme_observations_vs_oracle(md, kind, dtype):
    """All-zero frames (every pixel on the floor), saturated frames and salt-and-pepper impulse
    noise (the robust data term's case, deconv.py:142-180) match the oracle."""
    psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 9)
    params = md.DeconvParams()
    g = md.make_test_image(64, 128)
    if kind == "zeros":
        f = np.zeros((64, 128))
    elif kind == "saturated":
        f = np.full((64, 128), 255.0)
    else:
        f = md.synth_blur(g, psf).values.copy()
        rng = np.random.default_rng(4)
        hit = rng.random(f.shape) < 0.05
        f[hit] = np.where(rng.random(hit.sum()) < 0.5, 0.0, 255.0)
    out = md.DeblurPipeline(f.shape, psf, params, md.Scenario.BOX_1D, dtype=dtype).run(md.Image(f)).values
    ref = _oracle(md, f, psf, params, "box")
    assert np.isfinite(out).all()
    assert np.abs(out - ref).max() <= TOL


def test_longest_lines_vs_oracle(md):
    """The longest float32 blur axes: 4096-sample lines through Wiener + RRRL (the line-iteration
    kernel's on-chip limit) and 8192-sample lines through the Wiener step alone (the line FFT's)."""
    psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15)
    for n, iters in ((4096, 2), (8192, 0)):
        params = md.DeconvParams(iterations=iters)
        g = md.make_test_image(n, 16)
        f = md.quantize(md.add_gaussian_noise(md.synth_blur(g, psf), 5.0, seed=2)).values
        out = md.DeblurPipeline(f.shape, psf, params, dtype="float32").run(md.Image(f)).values
        ref = _oracle(md, f, psf, params, "box")
        assert np.abs(out - ref).max() <= TOL, n


@pytest.mark.parametrize("shape,axis,dtype,iters,scenario", [
    ((16, 16384), "h", "float32", 2, "BOX_1D"),       # past the f32 line FFT (8192)
    ((16, 8192), "h", "float32", 3, "BOX_1D"),        # past the f32 line-iteration kernel (4096)
    ((4096, 16), "v", "float64", 2, "BOX_1D"),        # past the f64 line-iteration kernel (2048)
    ((8192, 16), "v", "float64", 1, "BOX_1D"),        # past the f64 line FFT (4096)
    ((16, 16384), "h", "float32", 2, "FOURIER_1D"),   # periodic along the blur axis
    ((12, 16384), "h", "float32", 0, "BOX_1D"),       # cross axis not a power of two (fft.py:63-66
    ((12, 8192), "h", "float64", 2, "BOX_1D"),        #   constrains the blur axis only)
    ((8192, 20), "v", "float64", 2, "FOURIER_1D"),
    ((3, 65536), "h", "float64", 1, "BOX_1D"),        # a long line: two-level 1D transform
])
def test_lines_beyond_chip_as_plane(md, shape, axis, dtype, iters, scenario):
    """Blur axes longer than the on-chip line kernels take run as a plane with a one-row (one-
    column) PSF -- two-level FFT Wiener, direct-tap iterations with the line path's boundary --
    and still match the oracle's line pipeline."""
    ax = md.BlurAxis.HORIZONTAL if axis == "h" else md.BlurAxis.VERTICAL
    psf = md.Psf.uniform_box(ax, 15)
    params = md.DeconvParams(iterations=iters)
    g = md.Image(md.make_test_image(max(16, shape[1]), max(16, shape[0])).values[:shape[0], :shape[1]])
    assert g.values.shape == shape
    f = md.quantize(md.add_gaussian_noise(md.synth_blur(g, psf), 5.0, seed=3)).values
    pipe = md.DeblurPipeline(f.shape, psf, params, scenario=getattr(md.Scenario, scenario), dtype=dtype)
    assert pipe._plan.describe.startswith("1D PSF beyond the on-chip line limits as a plane"), pipe._plan.describe
    out = pipe.run(md.Image(f)).values
    ref = _oracle(md, f, psf, params, "box" if scenario == "BOX_1D" else "fourier1d")
    assert np.abs(out - ref).max() <= TOL, (shape, dtype)


def test_limits_raise(md):
    """Blur axes that are not powers of two raise ValueError at plan creation, short or long
    (the reference's own ValueError cases, fft.py:63-66)."""
    psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15)
    for shape, dtype, iters in (((16, 100), "float64", 5), ((12, 12288), "float32", 0),
                                ((12, 8200), "float64", 2)):
        with pytest.raises(ValueError):
            md.DeblurPipeline(shape, psf, md.DeconvParams(iterations=iters), dtype=dtype)


def test_one_plan_from_two_threads_and_streams(md):
    """A plan used concurrently from two host threads on two CUDA streams (ctypes releases the
    GIL): the per-plan lock serialises the enqueue, and a call on another stream waits for the
    previous one on the device (shared scratch), so every result equals the sequential one."""
    import threading
    import torch
    psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15)
    pipe = md.DeblurPipeline((256, 256), psf, md.DeconvParams(), dtype="float32")
    g = md.make_test_image(256, 256)
    base = torch.from_numpy(md.synth_blur(g, psf).values).float().cuda()
    batches = [base[None].repeat(64, 1, 1) + float(i) for i in range(6)]
    want = [pipe.run_batch(b).clone() for b in batches]
    torch.cuda.synchronize()
    outs = [torch.empty_like(b) for b in batches]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]

    def worker(k):
        with torch.cuda.stream(streams[k]):
            for i in range(k, len(batches), 2):
                pipe.plan.run(batches[i], out=outs[i], stream=streams[k])

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    torch.cuda.synchronize()
    for o, w in zip(outs, want):
        assert torch.equal(o, w)


def test_bench_pipeline_stage_samples(md):
    """bench_pipeline (bench.py:80-115) on CUDA-event stage times: stage names, pooled iteration
    samples (runs x iterations), first / later split, positive times; report renders them."""
    psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 9)
    f = md.synth_blur(md.make_test_image(64, 64), psf)
    for dtype in ("float64", "float32"):
        st = md.bench_pipeline(f, psf, md.DeconvParams(), runs=3, warmup=True, split_first_iteration=True, dtype=dtype)
        assert st.runs == 3
        assert list(st.per_stage) == ["wiener", "rrrl_iteration", "rrrl_total", "total", "rrrl_first_iteration",
                                      "rrrl_later_iterations"]
        assert st.per_stage["rrrl_iteration"].samples == 15
        assert st.per_stage["rrrl_later_iterations"].samples == 12
        assert st.mean_ms > 0 and st.per_stage["wiener"].mean_ms > 0
        assert md.report(st, "csv").startswith("scenario,stage,runs,mean_ms,std_ms,min_ms,max_ms\n")


# The per-iteration 2D-PSF stage kernels load their u tiles by TMA (md_tma.cuh) where the
# tensor map can be made, the rest per element: boxes must start on 16-byte column boundaries
# (an odd left halo shifts the tile inside its shared-memory row), frames whose row pitch is not
# a multiple of 16 bytes take the per-element path, and edge tiles of stage A wrap / clamp per
# element while interior tiles arrive by TMA. Every combination against the oracle.
def _tile_psf(md, kind):
    if kind == "line_odd":
        return md.Psf.line(9.0, 30.0)
    if kind == "line_even":
        return md.Psf.line(12.0, 75.0)
    w = np.random.default_rng(11).uniform(0.2, 1.0, size=(4, 5))
    return md.Psf.general_2d(w / w.sum(), center=(1, 3))


def _tile_input(md, shape, psf):
    g = md.make_test_image(shape[1], shape[0], seed=3)          # (width, height)
    return md.quantize(md.add_gaussian_noise(md.synth_blur(g, psf), 5.0, seed=4)).values


@pytest.mark.parametrize("shape", [(64, 64), (128, 256), (256, 512)])
@pytest.mark.parametrize("psf_kind", ["line_odd", "line_even", "small2d"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_plane_tile_loads_periodic_vs_oracle(md, shape, psf_kind, dtype):
    psf = _tile_psf(md, psf_kind)
    f = _tile_input(md, shape, psf)
    params = md.DeconvParams(iterations=3)
    pipe = md.DeblurPipeline(shape, psf, params, md.Scenario.FOURIER_2D, dtype=dtype, fused=False)
    assert "direct taps" in pipe.plan.describe and "fused" not in pipe.plan.describe
    out = pipe.run(md.Image(f)).values
    ref = _oracle(md, f, psf, params, "fourier2d")
    err = float(np.abs(out - ref).max())
    assert err <= (1e-6 if dtype == "float64" else TOL), err


@pytest.mark.parametrize("shape", [(96, 192), (128, 136), (130, 130), (200, 264), (72, 300)])
@pytest.mark.parametrize("psf_kind", ["line_odd", "small2d"])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_plane_tile_loads_clamped_vs_oracle(md, shape, psf_kind, dtype):
    from oracle import wr3l_oracle as O
    psf = _tile_psf(md, psf_kind)
    f = _tile_input(md, shape, psf)
    params = md.DeconvParams(iterations=3)
    out = md.rrrl_deblur(md.Image(f), psf, params, convolver="spatial", dtype=dtype).values
    p = O.OParams(wiener_k=params.wiener_k, alpha=params.alpha, iterations=params.iterations,
                  eps_data=params.eps_data, eps_reg=params.eps_reg, floor=params.floor)
    ref = O.rrrl_deblur(np.asarray(f, dtype=np.float64), O.OPsf("2d", psf.weights, psf.center), p, mode="spatial")
    err = float(np.abs(out - ref).max())
    assert err <= (1e-6 if dtype == "float64" else TOL), err
