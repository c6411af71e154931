#!/usr/bin/env python
"""Throughput benchmark of the Wiener + RRRL path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c1|c4] [--dtype float32|float64] [--batch B]

One "step" = the whole pipeline (Wiener init + RRRL iterations) over one batch of B
synthetic 256x256 frames resident in HBM. ``value`` = frames/s over all ranks (weak scaling:
B frames per GPU per step; frames are independent -- no collective on the data path), timed
with CUDA events, max over ranks. ``e2e`` = the same metric through the public host-buffer
entry (DeblurPipeline.run_batch on pinned host arrays -> md_run_host_ex: H2D + run + D2H
inside the timed region). ``--impl reference`` times the reference algorithm (the CPU
oracle port, oracle/wr3l_oracle.py) on all host cores: the CPU-baseline arm.

Workloads:
  c1  256x256, uniform horizontal box L=15, Gaussian noise sigma=5, Wiener + 5 RRRL
      (BASELINE.json configs[0]: the metric's 256^2 Wiener+RRRL frame). Default.
  c4  256x256 frames over a bank of 48 PSFs: 16 uniform boxes (H/V, L in [5,31] incl.
      fractional), 16 axis-aligned general 1D kernels, 16 2D kernels (12 lines at random
      angles, L<=21, + 4 small dense kernels); sigma=5, Wiener + 5 RRRL (configs[3]).
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "deblurred frames/sec (256² Wiener+RRRL) per GPU & 8 GPUs; p50 ms/frame; % HBM roofline"
H = W = 256
PX = H * W


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


def measured_traffic(key: str, frames: int):
    """DRAM bytes of the dominant kernel for `frames` frames per launch, scaled from the
    committed ncu capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            d = json.load(fh)[key]
        return (d["dram_bytes_read"] + d["dram_bytes_write"]) / d["frames"] * frames
    except Exception:
        return None


def measured_smem(key: str, frames: int):
    """Shared-memory wavefronts (128 B) of the dominant kernel for `frames` frames, from the
    committed ncu capture, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            d = json.load(fh)[key]
        return d["smem_wavefronts"] / d["frames"] * frames
    except Exception:
        return None


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def noisy(blurred: np.ndarray, seed: int, sigma: float = 5.0) -> np.ndarray:
    """quantize(add_gaussian_noise(., sigma, seed)) of synth.py:29-55 (PCG64)."""
    n = blurred + np.random.default_rng(seed).normal(0.0, sigma, blurred.shape)
    return np.clip(np.floor(np.clip(n, 0.0, 255.0) + 0.5), 0.0, 255.0)


# ---------------------------------------------------------------------------------- workloads
#
# A workload is built in two halves: the INPUTS (host NumPy: the deterministic scene, the
# blur, PCG64 noise) and, for the GPU arm only, the PIPELINE. The reference arm builds its
# inputs with the CPU oracle's clamped convolution (bit-identical to the GPU synth kernel,
# tests/test_gpu_parity.py) and never touches the device or libmdcuda.so.

def gpu_synth(md):
    return lambda g, psf: md.synth_blur(md.Image(g), psf).values


def cpu_synth(md):
    def blur(g, psf):
        return np.clip(np.floor(O_clamped(g, oracle_spec(psf)) + 0.5), 0.0, 255.0)
    return blur


def O_clamped(g, spec):
    from oracle import wr3l_oracle as O
    return O.clamped_convolve(np.asarray(g, dtype=np.float64), spec)


class C1:
    """configs[0]: 256^2, horizontal box L=15, sigma=5, Wiener + 5 RRRL."""

    name = "c1: 256x256 box L=15 horizontal, sigma=5, Wiener + 5 RRRL (BASELINE.json configs[0])"
    profile_in_loop = True                     # stage marks on the same stream cost nothing here

    def __init__(self, md, args, synth, gpu: bool = True):
        self.md = md
        self.psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15)
        self.params = md.DeconvParams()
        blurred = synth(md.make_test_image(W, H, seed=7).values, self.psf)
        k = min(64, args.batch)
        base = np.stack([noisy(blurred, 5 + i) for i in range(k)])
        self.host = np.tile(base, (-(-args.batch // k), 1, 1))[:args.batch]
        self.cpu_items = [("box", self.psf, base[i]) for i in range(k)]
        if gpu:
            self.pipe = self.make_pipe(args.dtype, args.fused)
            self.describe = self.pipe.plan.describe
            self.fused = self.pipe.plan.fused
            self.latency_plan = self.pipe.plan

    def make_pipe(self, dtype, fused="auto"):
        fz = None if fused == "auto" else fused == "on"
        pipe = self.md.DeblurPipeline((H, W), self.psf, self.params, self.md.Scenario.BOX_1D, dtype=dtype, fused=fz)
        if os.environ.get("MD_C1_CHUNK"):                 # measurement knob: frames per pipelined chunk
            pipe.plan.set_chunk(int(os.environ["MD_C1_CHUNK"]))
        return pipe

    def frames_per_iter_launch(self, n) -> float:
        """Frames one launch of the iteration kernel covers: the fused kernel runs every
        iteration of a chunk in one launch, the per-iteration kernel one launch per iteration
        (md_run_launch_count = chunks x (1 Wiener + iteration launches))."""
        per_chunk = 2 if self.fused else 1 + self.params.iterations
        return n / max(1, self.pipe.plan.launch_count(n) // per_chunk)

    def run(self, f, u):
        self.pipe.plan.run(f, out=u)

    @staticmethod
    def e2e_entry(src, dst) -> str:
        return f"DeblurPipeline.run_batch({src}) -> {dst} (md_run_host_ex, copies pipelined over 3 streams)"

    def run_profile(self, f, u) -> dict:
        return self.pipe.plan.run_profile(f, out=u)

    def e2e_set(self, nb):
        return self.host[:nb], None

    def device_frames(self, dtype):
        import torch
        return torch.from_numpy(self.host).to(device="cuda", dtype=dtype).contiguous()

    def run_host(self, hin, hout, ctx):
        self.pipe.run_batch(hin, out=hout, out_dtype=hout.dtype)

    def launches(self, n) -> int:
        return self.pipe.plan.launch_count(n)

    def iter_bytes(self, n, esz) -> float:
        """SURVEY 8(d) algorithmic bytes of the iteration stage for n frames (8 passes/it.)."""
        return 8 * self.params.iterations * PX * esz * n

    def frame_bytes(self, esz) -> float:
        """SURVEY 8(d) algorithmic bytes of one whole frame (Wiener-1D 2 passes + 8 per it.)."""
        return (2 + 8 * self.params.iterations) * PX * esz


def c4_bank(md, seed: int = 2026):
    """48 PSFs: 16 boxes, 16 general 1D, 16 2D (12 lines + 4 small dense kernels)."""
    rng = np.random.default_rng(seed)
    bank, kinds = [], []
    for i in range(16):
        axis = md.BlurAxis.HORIZONTAL if i % 2 == 0 else md.BlurAxis.VERTICAL
        L = float(rng.integers(5, 32)) + (0.5 if i % 4 == 3 else 0.0)
        bank.append(md.Psf.uniform_box(axis, min(L, 31.0)))
        kinds.append("box")
    for i in range(16):
        axis = md.BlurAxis.HORIZONTAL if i % 2 == 0 else md.BlurAxis.VERTICAL
        taps = int(rng.integers(5, 18))
        w = np.exp(-np.linspace(0.0, rng.uniform(0.5, 3.0), taps)) * rng.uniform(0.5, 1.0, taps)
        bank.append(md.Psf.general_1d(w, axis, center=int(rng.integers(taps // 3, 2 * taps // 3 + 1))))
        kinds.append("fourier1d")
    for i in range(16):
        if i < 12:
            bank.append(md.Psf.line(float(rng.uniform(7.0, 21.0)), float(rng.uniform(0.0, 180.0))))
        else:
            s = int(rng.integers(3, 8))
            bank.append(md.Psf.general_2d(rng.uniform(0.0, 1.0, (s, s))))
        kinds.append("fourier2d")
    return bank, kinds


C4_SCENE_SEEDS = (7, 8, 9, 10)
# PSF groups dealt round-robin over CUDA streams in the timed c4 step (PsfBankPipeline.run): 3
# measured 0.7 % faster than 2 at 65536 frames; groups by class (2D tile kernels on their own
# stream beside the cluster kernels) 0.5 % slower (scripts/c4_deal_ab.sh)
C4_STREAMS = int(os.environ.get("MD_C4_STREAMS", "3"))


C4_DISTINCT = 8                      # distinct noisy frames per PSF (4 scenes x 2 noise draws)


def c4_distinct(md, bank, synth, used=None):
    """[len(bank), C4_DISTINCT, H, W]: the distinct noisy frames of every PSF in `used` (default all;
    the others stay zero) -- 8 per PSF over the 4 scenes, noise seeded by (PSF, frame)."""
    scenes = [md.make_test_image(W, H, seed=s).values for s in C4_SCENE_SEEDS]
    out = np.zeros((len(bank), C4_DISTINCT, H, W))
    for b, psf in enumerate(bank):
        if used is not None and b not in used:
            continue
        blurred = [synth(scenes[j], psf) for j in range(4)]
        out[b] = np.stack([noisy(blurred[j % 4], 1000 * b + j) for j in range(C4_DISTINCT)])
    return out


def c4_source(index):
    """Frame i (PSF index[i], k-th frame of its PSF) is distinct frame (index[i], k mod 8)."""
    idx = np.asarray(index)
    k = np.zeros(idx.size, dtype=np.int64)
    for b in np.unique(idx):
        sel = np.nonzero(idx == b)[0]
        k[sel] = np.arange(sel.size)
    return idx * C4_DISTINCT + k % C4_DISTINCT


def c4_frames(md, bank, index, synth, with_scenes=False):
    """The c4 frames for PSF assignment `index` (8 distinct noisy frames per PSF, 4 scenes),
    plus one (kind, psf, frame) CPU sample item per PSF [and each frame's scene number]."""
    used = set(int(b) for b in np.unique(index))
    base = c4_distinct(md, bank, synth, used).reshape(-1, H, W)
    src = c4_source(index)
    frames = base[src]
    scene_of = (src % C4_DISTINCT) % 4
    items = [(b, bank[b], base[b * C4_DISTINCT]) for b in sorted(used)]
    return (frames, items, scene_of) if with_scenes else (frames, items)


class C4:
    """configs[3]: 256^2 frames over a 48-PSF bank, grouped by PSF."""

    name = ("c4: 256x256 frames, 48-PSF bank (16 box H/V L 5-31 incl. fractional, 16 general 1D, "
            "12 lines L<=21 at random angles + 4 small 2D), sigma=5, Wiener + 5 RRRL (BASELINE.json configs[3])")
    # the timed step deals the PSF groups over two streams (one group's last partial cluster
    # wave overlaps the next group); the stage split comes from a separate, sequential pass
    profile_in_loop = False

    def __init__(self, md, args, synth, gpu: bool = True):
        self.md = md
        self.params = md.DeconvParams()
        self.bank, self.kinds = c4_bank(md)
        nb = len(self.bank)
        # strong scaling (configs[3], the default): ONE batch of args.global_batch frames over the
        # ranks, rank r taking frames r, r + N, ... (every rank sees every PSF class); weak (an
        # explicit --batch): args.batch frames per rank
        gb = getattr(args, "global_batch", None)
        G = gb or args.batch
        per = -(-G // nb)
        gidx = np.minimum(np.arange(G) // per, nb - 1)
        gsrc = c4_source(gidx)
        sel = slice(getattr(args, "rank", 0), None, getattr(args, "world", 1)) if gb else slice(None)
        self.index, self.src = gidx[sel], gsrc[sel]
        assert self.index.size == args.batch, (self.index.size, args.batch)
        self.distinct = c4_distinct(md, self.bank, synth).reshape(-1, H, W)
        self.cpu_items = [(self.kinds[b], psf, self.distinct[b * C4_DISTINCT]) for b, psf in enumerate(self.bank)]
        if gpu:
            from paper_1212_2245_b200.batch import PsfBankPipeline
            self.pipe = PsfBankPipeline((H, W), self.bank, self.params, dtype=args.dtype)
            self.describe = "; ".join(sorted({p.plan.describe.split(",")[0] for p in self.pipe.pipes}))
            self.fused = False
            self.latency_plan = self.pipe.pipes[int(self.index[0])].plan

    def device_frames(self, dtype):
        """The rank's frames in HBM, gathered on the device from the distinct ones."""
        import torch
        d = torch.from_numpy(self.distinct).to(device="cuda", dtype=dtype)
        return d[torch.from_numpy(self.src).cuda()].contiguous()

    def make_pipe(self, dtype, fused="auto"):
        from paper_1212_2245_b200.batch import PsfBankPipeline
        return PsfBankPipeline((H, W), self.bank, self.params, dtype=dtype)

    def run(self, f, u, pipe=None, index=None):
        (pipe or self.pipe).run(f, self.index if index is None else index, out=u, streams=C4_STREAMS)

    def run_profile(self, f, u) -> dict:
        tot = {"init_ms": 0.0, "iter_ms": 0.0, "layout_ms": 0.0, "groups": 0}
        for b, s, e in self.pipe.groups(self.index):
            p = self.pipe.pipes[b].plan.run_profile(f[s:e], out=u[s:e])
            for k in tot:
                tot[k] += p[k]
        return tot

    def e2e_set(self, nb):
        sel = np.linspace(0, self.index.size - 1, nb).astype(np.int64)   # every PSF class, sorted
        return self.distinct[self.src[sel]], self.index[sel]

    def run_host(self, hin, hout, ctx):
        self.pipe.run_host(hin, ctx, out=hout)

    @staticmethod
    def e2e_entry(src, dst) -> str:
        return (f"PsfBankPipeline.run_host({src}) -> {dst} (copies of PSF group g+1 / g-1 overlap the "
                "deconvolution of group g: 3 streams, md_convert + md_run per group)")

    def launches(self, n) -> int:
        return self.pipe.launch_count(self.index[:n])

    def frames_per_iter_launch(self, n):
        return None                            # many kernels per step: no single dominant launch

    def iter_bytes(self, n, esz) -> float:
        # 8 passes per iteration for every class (line / box / direct-tap convolvers)
        return 8 * self.params.iterations * PX * esz * n

    def frame_bytes(self, esz) -> float:
        return (2 + 8 * self.params.iterations) * PX * esz


class Single:
    """configs[1] / configs[2]: one large frame geometry with one 2D PSF, a batch of frames per
    step through one DeblurPipeline (FOURIER_2D: direct taps for the line PSF, the 2D-FFT
    convolver for the dense 31x31 one). Noise-free inputs, as SURVEY 8(d) states them."""

    profile_in_loop = True
    fused = False
    cpu_frames_per_core = 1

    def __init__(self, md, args, synth, gpu: bool = True):
        self.md = md
        self.params = md.DeconvParams(iterations=self.iterations)
        self.psf = self.make_psf(md)
        n = self.side
        base = np.stack([synth(md.make_test_image(n, n, seed=s).values, self.psf) for s in (7, 8, 9, 10)])
        self.base = base
        self.src = np.arange(args.batch) % base.shape[0]
        self.cpu_items = [("fourier2d", self.psf, base[i]) for i in range(base.shape[0])]
        if gpu:
            self.pipe = self.make_pipe(args.dtype)
            self.describe = self.pipe.plan.describe
            self.latency_plan = self.pipe.plan

    def make_pipe(self, dtype, fused="auto"):
        return self.md.DeblurPipeline((self.side, self.side), self.psf, self.params, self.md.Scenario.FOURIER_2D,
                                      dtype=dtype)

    def device_frames(self, dtype):
        import torch
        d = torch.from_numpy(self.base).to(device="cuda", dtype=dtype)
        return d[torch.from_numpy(self.src).cuda()].contiguous()

    def run(self, f, u):
        self.pipe.plan.run(f, out=u)

    def run_profile(self, f, u) -> dict:
        return self.pipe.plan.run_profile(f, out=u)

    def e2e_set(self, nb):
        return self.base[self.src[:nb]], None

    def run_host(self, hin, hout, ctx):
        self.pipe.run_batch(hin, out=hout, out_dtype=hout.dtype)

    @staticmethod
    def e2e_entry(src, dst) -> str:
        return f"DeblurPipeline.run_batch({src}) -> {dst} (md_run_host_ex, copies pipelined over 3 streams)"

    def launches(self, n) -> int:
        return self.pipe.plan.launch_count(n)

    def frames_per_iter_launch(self, n):
        return None

    def iter_bytes(self, n, esz) -> float:
        return self.passes_per_iteration * self.params.iterations * self.side ** 2 * esz * n

    def frame_bytes(self, esz) -> float:
        return (7 + self.passes_per_iteration * self.params.iterations) * self.side ** 2 * esz


class C2(Single):
    name = ("c2: 512x512 line PSF L=21 @30 deg (sub-pixel, 63 taps), noise-free, Wiener + 10 RRRL, direct taps "
            "(BASELINE.json configs[1])")
    side, iterations, batch = 512, 10, 256
    metric = "c2: deblurred 512^2 frames/s (line PSF, Wiener + 10 RRRL); % HBM roofline"
    passes_per_iteration = 8            # line direct = 7 + 10 x 8 field passes per frame
    cpu_frames_per_core = 2

    @staticmethod
    def make_psf(md):
        return md.Psf.line(21.0, 30.0)


class C3(Single):
    name = ("c3: 1024x1024 dense 31x31 PSF exp(-r^2/50) x U(0.2, 1) (seed 3), noise-free, 2D-FFT Wiener + 5 RRRL "
            "(BASELINE.json configs[2])")
    side, iterations, batch = 1024, 5, 64
    metric = "c3: deblurred 1024^2 frames/s (dense 31x31 PSF, 2D-FFT Wiener + 5 RRRL); % HBM roofline"
    passes_per_iteration = 18           # 2D-FFT convolver = 7 + 5 x 18 field passes per frame

    @staticmethod
    def make_psf(md):
        yy, xx = np.mgrid[-15:16, -15:16]
        return md.Psf.general_2d(np.exp(-(yy ** 2 + xx ** 2) / 50.0) * np.random.default_rng(3).uniform(0.2, 1.0, (31, 31)))


WORKLOADS = {"c1": C1, "c2": C2, "c3": C3, "c4": C4}


def bench_config(work_name: str, batch: int, world: int, esz: int, global_batch=None) -> dict:
    """The `config` object both arms print (identical for the same command line)."""
    c = {"workload": work_name, "frames_per_gpu_per_step": batch, "parallelism": f"frame-sharded x{world}",
         "l2": f"inputs {batch * PX * esz / 2**20:.0f} MiB per GPU > 126 MB L2 (no reuse between steps)"}
    if global_batch:
        c["global_batch"] = global_batch
        c["parallelism"] = f"one {global_batch}-frame batch, frames dealt round-robin over {world} rank(s)"
    return c


def run_c5(args, rank: int, world: int, local: int) -> None:
    """configs[4]: ONE size x size image (default 16384^2), line L=21 @30 deg, float64,
    Wiener + 5 RRRL. N=1: the whole image through one plan (two-level FFT Wiener, direct-tap
    iterations). N>1: row slabs over the ranks, NCCL halo exchange and all-to-all spectrum
    transposes (paper_1212_2245_b200/slab.py). Metric: images/s (and Mpx/s); SURVEY 8(d)
    algorithmic bytes per image = (7 + 5*8) field passes x 8 B x px."""
    import torch
    import torch.distributed as dist
    import paper_1212_2245_b200 as md
    from paper_1212_2245_b200.slab import CudaSlabBackend, DistComm, SlabGeometry, SlabWorker
    n = args.size
    psf = md.Psf.line(21.0, 30.0)
    params = md.DeconvParams()
    gen = torch.Generator(device="cuda").manual_seed(5)
    # synthetic scene on the device: smooth gradient + random blocks, blurred (clamped, GPU), 8-bit
    yy = torch.linspace(0, 1, n, device="cuda", dtype=torch.float64)
    g = 60.0 + 100.0 * yy[:, None] + 60.0 * yy[None, :]
    blocks = torch.rand((n // 64, n // 64), generator=gen, device="cuda", dtype=torch.float64)
    g = g + 40.0 * (blocks.repeat_interleave(64, 0).repeat_interleave(64, 1) - 0.5)
    conv = md.make_convolver(psf, (n, n), "spatial")
    f = torch.clamp(torch.floor(conv.blur(g.contiguous()) + 0.5), 0, 255)
    del g
    pipe = md.DeblurPipeline((n, n), psf, params, big_fft=True)
    stream = torch.cuda.current_stream()
    if world == 1:
        u = torch.empty_like(f)
        run = lambda: pipe.plan.run(f, out=u)
    else:
        be = CudaSlabBackend(pipe.plan)
        geo = SlabGeometry(n, n, rank, world, *be.halo_rows())
        worker = SlabWorker(be, geo, params.iterations, f.device, f.dtype)
        comm = DistComm()
        S = n // world
        f_own = f[rank * S:(rank + 1) * S].contiguous()
        del f
        run = lambda: worker.run(comm, f_own)
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            run()
        ev1.record(stream)
        torch.cuda.synchronize()
    t = torch.tensor([ev0.elapsed_time(ev1)], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    e2e = None
    if world == 1:
        # end to end through the public host entry: the pinned 8-bit image in (the synthetic
        # input is quantised to 8 bits, like the c1 / c4 e2e frames), float64 out
        # (DeblurPipeline.run_batch(ndarray) -> md_run_host_ex), copies inside the timed region
        q = f.round().clamp(0, 255)
        assert bool(torch.equal(q, f)), "c5 input is not 8-bit quantised"
        hin = q.to(torch.uint8).cpu().pin_memory()
        hout = torch.empty(hin.shape, dtype=torch.float64).pin_memory()
        hin_np, hout_np = hin.numpy(), hout.numpy()
        pipe.run_batch(hin_np, out=hout_np)
        steps = max(2, min(5, args.steps))
        t0 = time.perf_counter()
        for _ in range(steps):
            pipe.run_batch(hin_np, out=hout_np)
        el = (time.perf_counter() - t0) / steps
        e2e = {"value": 1.0 / el, "unit": "images/s", "h2d_bytes_per_step": hin_np.nbytes,
               "d2h_bytes_per_step": hout_np.nbytes,
               "entry": "DeblurPipeline.run_batch(pinned uint8 image) -> float64 (md_run_host_ex)"}
    fp64 = None
    if world == 1:
        # the direct-tap iterations are FP64-ALU work: their flops against a measured FP64 peak
        # (cuBLAS DGEMM here, the same data path as the FP64 FMA units on B200)
        prof = pipe.plan.run_profile(f, out=u)
        taps = int(np.count_nonzero(psf.weights))
        flops = 2.0 * 3 * taps * n * n * params.iterations
        a = torch.randn((8192, 8192), device="cuda", dtype=torch.float64)
        for _ in range(2):
            a @ a
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            a @ a
        e1.record()
        e1.synchronize()
        peak_tf = 3 * 2 * 8192.0 ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12
        del a
        ach = flops / (prof["iter_ms"] / 1e3) / 1e12
        fp64 = {"bound": "fp64", "kernel": "direct-tap RRRL iteration stages (k_plane_a_fast / k_plane_b_fast)",
                "achieved": ach, "peak": peak_tf, "unit": "TFLOP/s", "frac": ach / peak_tf,
                "peak_source": "measured in this run: cuBLAS DGEMM 8192^3 (torch.matmul float64)",
                "flop_model": f"2 flop x (blur + adjoint pair = 3) x {taps} taps per pixel per iteration",
                "stage_ms": {k: prof[k] for k in ("init_ms", "iter_ms")}}
    if rank == 0:
        pk = peaks()
        bytes_img = (7 + 8 * params.iterations) * 8 * n * n
        line = {
            "metric": "c5: single-image deblur throughput (images/s)", "value": 1e3 / ms, "unit": "images/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device-generated scene, GPU clamped line blur, 8-bit)",
            "config": {"workload": f"c5: one {n}x{n} image, line L=21 @30deg, Wiener + 5 RRRL (BASELINE.json "
                                   "configs[4])", "parallelism": f"row slabs x{world}" if world > 1 else "one plan",
                       "plan": pipe.plan.describe},
            "mpx_per_s": n * n / ms / 1e3,
            "roofline": {"bound": "hbm", "kernel": "whole pipeline", "achieved": bytes_img / (ms / 1e3) / 1e9 / world,
                         "peak": pk["hbm_gbs"], "unit": "GB/s per GPU",
                         "frac": bytes_img / (ms / 1e3) / 1e9 / world / pk["hbm_gbs"], "traffic": None,
                         "bytes_model": "SURVEY.md 8(d): (7 + 5x8) field passes x 8 B per pixel"},
            "roofline_fp64": fp64,
            "gpu_launches": pipe.plan.launch_count(1) * args.steps if world == 1 else None,
            "cpu_baseline": None,
            "e2e": e2e,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.stamps, self.proc = index, [], [], None
        self.t_start = self.t_end = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0:   # first sample before timing starts
                time.sleep(0.02)
        except Exception:
            self.proc = None
        self.t_start = time.time()
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)
                self.stamps.append(time.time())

    def __exit__(self, *exc):
        self.t_end = time.time()
        time.sleep(0.25)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        rows = [r for r, t in zip(self.rows, self.stamps)
                if self.t_start is not None and self.t_start <= t <= (self.t_end or t) + 0.2]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [v for v in (num(r[0]) for r in rows) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": num(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------------- CPU arm

def _cpu_worker(job):
    """Time the oracle port of the reference pipeline on a list of (kind, psf-spec, frame)."""
    from oracle import wr3l_oracle as O
    t0 = time.perf_counter()
    for kind, spec, f, iters in job:
        O.pipeline(f, spec, O.OParams(iterations=iters), kind)
    return time.perf_counter() - t0


def oracle_spec(psf):
    from oracle import wr3l_oracle as O
    if psf.kind.value == "box":
        return O.OPsf("box", np.asarray(psf.weights), int(psf.center), psf.axis.value, float(psf.length))
    if psf.kind.value == "1d":
        return O.OPsf("1d", np.asarray(psf.weights), int(psf.center), psf.axis.value)
    return O.OPsf("2d", np.asarray(psf.weights), tuple(psf.center))


def cpu_jobs(work, per_core: int, cores: int):
    """Per-core frame lists with the workload's class mix."""
    iters = work.params.iterations
    items = [(k, oracle_spec(p), f, iters) for k, p, f in work.cpu_items]
    return [[items[(c * per_core + i) % len(items)] for i in range(per_core)] for c in range(cores)]


def cpu_rate(jobs, pool) -> tuple[float, float]:
    t0 = time.perf_counter()
    pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    return sum(len(j) for j in jobs) / wall, wall


def run_reference(args, rank: int, world: int) -> None:
    """--impl reference: the reference algorithm (the CPU oracle port of the reference's
    DeblurPipeline.run, NumPy float64) on all host cores. Inputs come from host NumPy and
    the oracle's clamped convolution: no device work, libmdcuda.so is never loaded.
    Under N>1 rank 0 alone runs; the other ranks exit without work."""
    if rank != 0:
        return
    import paper_1212_2245_b200 as md              # host-side value types only (Psf, scenes)
    esz = 8 if args.dtype == "float64" else 4       # only for the shared config object
    work = WORKLOADS[args.config](md, args, cpu_synth(md), gpu=False)
    cores = host_cores()
    jobs = cpu_jobs(work, args.cpu_frames_per_core, cores)
    pool = mp.get_context("fork").Pool(cores)
    for _ in range(args.warmup):
        cpu_rate(jobs, pool)
    walls = [cpu_rate(jobs, pool)[1] for _ in range(args.steps)]
    pool.close()
    pool.join()
    per_step = sum(len(j) for j in jobs)
    value = per_step * args.steps / sum(walls)
    sample = (f"{per_step} frames per step ({args.cpu_frames_per_core} per core) of this workload's frames "
              "through oracle/wr3l_oracle.pipeline (NumPy float64 restatement of the reference's "
              "DeblurPipeline.run: its radix-2 FFT and cumsum box filter), one process per host core")
    line = {
        "impl": "reference", "metric": getattr(work, "metric", METRIC), "value": value, "unit": "frames/s", "n_gpus": world,
        "devices": "host CPU cores only (n_gpus echoes the launch's N; no device work)",
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(walls) / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": DATA,
        "config": bench_config(work.name, args.batch, world, esz, args.global_batch),
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "p50_ms_per_frame": 1e3 * statistics.median(walls) / args.cpu_frames_per_core,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------- GPU arm

DATA = "synthetic (deterministic scenes, clamped-spatial blur, PCG64 sigma=5 noise, 8-bit)"


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1", choices=sorted(WORKLOADS) + ["c5"])
    ap.add_argument("--size", type=int, default=16384, help="c5 image side")
    ap.add_argument("--dtype", default="float64", choices=["float32", "float64"],
                    help="arithmetic of the timed path (default float64, the reference's: core.py:3-4)")
    ap.add_argument("--batch", type=int, default=None,
                    help="frames per GPU per step (weak scaling; c1 default 4096)")
    ap.add_argument("--global-batch", type=int, default=None,
                    help="c4: frames per step over ALL ranks (strong scaling; default 65536, configs[3])")
    ap.add_argument("--e2e-batch", type=int, default=2048)
    ap.add_argument("--cpu-frames-per-core", type=int, default=None,
                    help="CPU sample frames per host core (default: 24 for c1 / c4, 2 for c2, 1 for c3)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip latency / extra e2e / f32 context legs")
    ap.add_argument("--fused", default="auto", choices=["auto", "on", "off"])
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N>1 (gloo: CPU tests of the timing path)")
    args = ap.parse_args(argv)
    args.world = int(os.environ.get("WORLD_SIZE") or args.gpus)
    args.rank = int(os.environ.get("RANK", "0"))
    if args.config != "c4":
        args.global_batch = None
    elif args.batch is None and args.global_batch is None:
        args.global_batch = 65536
    if args.global_batch:
        if args.global_batch % args.world:
            ap.error(f"--global-batch {args.global_batch} does not split over {args.world} ranks")
        args.batch = args.global_batch // args.world
    elif args.batch is None:
        args.batch = WORKLOADS[args.config].batch if args.config in ("c2", "c3") else 4096
    if args.cpu_frames_per_core is None:
        args.cpu_frames_per_core = getattr(WORKLOADS.get(args.config), "cpu_frames_per_core", 24)
    args.scaling = "strong" if args.global_batch else "weak"
    return args


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawned(local: int, world: int, port: int, argv) -> None:
    os.environ.update({"RANK": str(local), "LOCAL_RANK": str(local), "WORLD_SIZE": str(world),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    rank_main(parse_args(argv))


def main(argv=None) -> None:
    args = parse_args(argv)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N` without torchrun: launch the N ranks here (one process per
        # GPU, RANK / LOCAL_RANK / WORLD_SIZE as torchrun would set them)
        import torch.multiprocessing as tmp
        port = _free_port()
        tmp.start_processes(_spawned, args=(args.gpus, port, sys.argv[1:] if argv is None else argv),
                            nprocs=args.gpus, join=True, start_method="spawn")
        return
    rank_main(args)


def rank_main(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    cuda = args.backend == "nccl"
    if cuda:
        torch.cuda.set_device(local)
    if world > 1:
        if cuda:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    try:
        if args.config == "c5":
            run_c5(args, rank, world, local)
        else:
            run_frames(args, rank, world, local, cuda)
    finally:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()


def timed_steps(run, steps: int, world: int, cuda: bool, stream=None, clk=None) -> float:
    """Time `steps` calls of run() after a barrier, CUDA events on the launching stream
    (synchronised on both sides); the max over ranks in ms."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    if cuda:
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(steps):
            run()
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
    else:
        t0 = time.perf_counter()
        for _ in range(steps):
            run()
        ms = (time.perf_counter() - t0) * 1e3
    t = torch.tensor([ms], dtype=torch.float64, device="cuda" if cuda else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_frames(args, rank: int, world: int, local: int, cuda: bool) -> None:
    """c1 / c4: B frames per GPU per step, frames independent (no collective on the data
    path); value = all ranks' frames / the max over ranks of the timed region."""
    import torch
    import torch.distributed as dist
    if not cuda:
        # CPU process-group test of the sharding / timing logic (tests/test_bench_dist.py):
        # the same barrier + max-over-ranks timing around a stand-in step, no device
        esz = 8 if args.dtype == "float64" else 4
        share = torch.zeros(args.batch, dtype=torch.float64)
        ms = timed_steps(lambda: share.add_(1.0), args.steps, world, False)
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": args.batch * args.steps * world / (ms / 1e3),
                              "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                              "ms_per_step": ms / args.steps, "backend": "gloo",
                              "config": bench_config(WORKLOADS[args.config].name, args.batch, world, esz, args.global_batch)}),
                  flush=True)
        return

    import paper_1212_2245_b200 as md
    work = WORKLOADS[args.config](md, args, gpu_synth(md))
    tdt = torch.float32 if args.dtype == "float32" else torch.float64
    esz = 4 if args.dtype == "float32" else 8
    f = work.device_frames(tdt)
    u = torch.empty_like(f)
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        work.run(f, u)
    torch.cuda.synchronize()
    prof = {"init_ms": 0.0, "iter_ms": 0.0, "layout_ms": 0.0, "groups": 0}

    def step():
        if work.profile_in_loop:
            p = work.run_profile(f, u)          # CUDA events between launch groups, same stream
            for k in prof:
                prof[k] += p[k]
        else:
            work.run(f, u)

    with ClockSampler(local) as clk:
        max_ms = timed_steps(step, args.steps, world, True, stream)
    if not work.profile_in_loop:
        # stage split from profiled sequential steps after the timed region, scaled to it
        npf = max(1, min(args.steps, 5))
        for _ in range(npf):
            p = work.run_profile(f, u)
            for k in prof:
                prof[k] += p[k] * args.steps / npf
    value = args.batch * args.steps * world / (max_ms / 1e3)

    extras = {}
    if not args.no_extras:
        # single-frame latency (p50 / p99 over 200 runs, batch = 1)
        f1, u1 = f[:1].clone(), torch.empty_like(f[:1])
        lat = []
        for i in range(210):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            work.latency_plan.run(f1, out=u1)
            b.record(stream)
            b.synchronize()
            if i >= 10:
                lat.append(a.elapsed_time(b))
        extras["p50_ms_per_frame_batch1"] = statistics.median(lat)
        extras["p99_ms_per_frame_batch1"] = sorted(lat)[min(len(lat) - 1, int(0.99 * len(lat)))]
        # host-observed single-frame latency (call -> result ready): direct md_run vs a replay
        # of the same run captured as a CUDA graph (GpuPlan.capture)
        g1 = work.latency_plan.capture(f1, u1)
        host_lat = {}
        for name, call in (("direct", lambda: work.latency_plan.run(f1, out=u1)), ("cuda_graph", g1.replay)):
            xs = []
            for i in range(110):
                t0 = time.perf_counter()
                call()
                torch.cuda.synchronize()
                if i >= 10:
                    xs.append((time.perf_counter() - t0) * 1e3)
            host_lat[name] = statistics.median(xs)
        del g1
        extras["host_p50_ms_per_frame_batch1"] = host_lat

    # end to end through the public host-buffer entry (DeblurPipeline.run_batch(ndarray) ->
    # md_run_host_ex): pinned host frames in, pinned host results out, copies inside the timed
    # region. Headline: the workload's native 8-bit frames in, float64 results out (the
    # reference's Image type, computed in float64).
    def e2e_rate(in_dtype, out_dtype, nb):
        frames, ctx = work.e2e_set(nb)
        hin = torch.from_numpy(np.ascontiguousarray(frames).astype(in_dtype)).pin_memory()
        hout = torch.empty(hin.shape, dtype=torch.from_numpy(np.zeros(1, out_dtype)).dtype).pin_memory()
        hin_np, hout_np = hin.numpy(), hout.numpy()
        work.run_host(hin_np, hout_np, ctx)
        torch.cuda.synchronize()
        steps = max(3, min(10, args.steps // 2))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            work.run_host(hin_np, hout_np, ctx)  # H2D + convert + run + convert + D2H, synchronous
        el = time.perf_counter() - t0
        te = torch.tensor([el], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        return {"value": nb * steps * world / float(te.item()), "unit": "frames/s",
                "h2d_bytes_per_step": hin_np.nbytes, "d2h_bytes_per_step": hout_np.nbytes, "frames_per_step": nb}

    nb = min(args.e2e_batch, args.batch)
    out_np = np.float64 if args.dtype == "float64" else np.float32
    e2e = e2e_rate(np.uint8, out_np, nb)
    e2e["entry"] = work.e2e_entry("pinned uint8 frames", f"{np.dtype(out_np).name} results, computed in {args.dtype}")
    if not args.no_extras:
        if args.dtype == "float64":
            x = e2e_rate(np.uint8, np.float32, nb)
            x["entry"] = work.e2e_entry("pinned uint8 frames", "float32 results (computed in float64, rounded "
                                        "on the device: half the PCIe bytes of the headline)")
            extras["e2e_f32_out"] = x
        x = e2e_rate(np.uint8, np.uint8, nb)
        x["entry"] = work.e2e_entry("pinned uint8 frames", "uint8 frames quantised like the reference's write_pgm "
                                    "(pgm.py:56-58), the CLI's output")
        extras["e2e_u8"] = x

    # context only, not the headline: the same frames through a float32 plan (the precision
    # SURVEY 8(d) measured safe for the noisy 256^2 configs; the reference computes in float64)
    f32_ctx = None
    if not args.no_extras and args.dtype == "float64":
        p32 = work.make_pipe("float32")
        # at most 16384 frames (every k-th: the same class mix), so the float32 copies fit beside
        # a large float64 batch
        k32 = max(1, args.batch // 16384)
        sel32 = torch.arange(0, args.batch, k32, device=f.device)
        n32 = int(sel32.numel())
        f32 = f[sel32].to(torch.float32)
        u32 = torch.empty_like(f32)
        if args.config == "c4":
            idx32 = work.index[::k32]
            run32 = lambda: work.run(f32, u32, pipe=p32, index=idx32)
        else:
            run32 = lambda: p32.plan.run(f32, out=u32)
        for _ in range(2):
            run32()
        ms32 = timed_steps(run32, max(3, args.steps // 2), world, True, stream)
        f32_ctx = {"value": n32 * max(3, args.steps // 2) * world / (ms32 / 1e3), "unit": "frames/s",
                   "dtype": "f32", "frames_per_gpu": n32,
                   "note": "context only: float32 arithmetic is narrower than the reference's"}
        del f32, u32, p32

    if rank == 0:
        pk = peaks()
        iter_bytes = work.iter_bytes(args.batch, esz) * args.steps
        iter_s = prof["iter_ms"] / 1e3
        achieved = iter_bytes / iter_s / 1e9 if prof["iter_ms"] > 0 else None
        cpu = None
        if not args.no_cpu and world == 1:            # the CPU baseline: rank 0 at N=1 only
            cores = host_cores()
            jobs = cpu_jobs(work, args.cpu_frames_per_core, cores)
            pool = mp.get_context("fork").Pool(cores)
            r, wall = cpu_rate(jobs, pool)
            pool.close()
            pool.join()
            cpu = {"value": r, "unit": "frames/s", "cores": cores, "kind": "port",
                   "sample": f"{sum(len(j) for j in jobs)} frames of this workload ({wall:.1f} s wall) through "
                             "oracle/wr3l_oracle.pipeline (NumPy float64), one process per host core"}
        key = f"{args.config}_{args.dtype}"
        fpl = work.frames_per_iter_launch(args.batch)
        traffic = measured_traffic(key, fpl) if fpl else None
        # the fused kernel keeps the iterate on chip, so its other roofline is the shared-memory
        # pipe (north_star: "HBM (or SMEM for fused in-cluster)"): ncu wavefronts per frame over
        # this run's iteration time, against SMs x 128 B/clk x the max SM clock
        smem_roof = None
        wf = measured_smem(key, args.batch) if work.fused else None
        if wf and prof["iter_ms"] > 0:
            sms = torch.cuda.get_device_properties(local).multi_processor_count
            ach = wf * 128 * args.steps / iter_s / 1e12
            pk_s = sms * 128 * pk["sm_max_mhz"] * 1e6 / 1e12
            smem_roof = {"bound": "smem", "kernel": "RRRL iteration (fused cluster kernel)", "achieved": ach,
                         "peak": pk_s, "unit": "TB/s", "frac": ach / pk_s,
                         "wavefronts_per_frame": wf / args.batch,
                         "source": "ncu l1tex__data_pipe_lsu_wavefronts_mem_shared.sum (profiles/ncu_traffic.json) "
                                   "over this run's iteration time; peak = SMs x 128 B/clk x max SM clock"}
        frame_gbs = value / world * work.frame_bytes(esz) / 1e9
        geom = work.pipe.plan.fused_geometry() if (work.fused and hasattr(work, "pipe")) else None
        if geom:
            geom["sms"] = torch.cuda.get_device_properties(local).multi_processor_count
        line = {
            "metric": getattr(work, "metric", METRIC), "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32" if args.dtype == "float32" else "f64",
            "data": DATA,
            "config": bench_config(work.name, args.batch, world, esz, args.global_batch),
            "plan": work.describe,
            **{k: v for k, v in extras.items() if not k.startswith("e2e")},
            "stage_ms_per_step": {k: prof[k] / args.steps for k in ("init_ms", "iter_ms", "layout_ms")},
            "stage_split_source": ("CUDA events between the launch groups of the timed steps" if work.profile_in_loop
                                   else "CUDA events of profiled sequential steps after the timed region"),
            "roofline": {"bound": "hbm",
                         "kernel": "RRRL iteration" + (" (fused cluster kernel)" if work.fused else " (per-iteration kernels)"),
                         "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": (achieved / pk["hbm_gbs"]) if achieved else None,
                         "traffic": traffic,
                         "traffic_note": "measured DRAM bytes per launch of the iteration kernel (ncu --set full, "
                                         "profiles/ncu_traffic.json, scaled to this launch's frames)",
                         "peak_source": pk["source"],
                         "bytes_model": "SURVEY.md 8(d): 8 field passes per RRRL iteration x 65536 px x "
                                        f"{esz} B per frame; time = CUDA events around the iteration launches",
                         "launch_geometry": geom},
            "roofline_frame": {"bound": "hbm", "achieved": frame_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                               "frac": frame_gbs / pk["hbm_gbs"],
                               "bytes_model": f"SURVEY.md 8(d): whole frame (Wiener 2 + 8 per iteration) field passes "
                                              f"x {esz} B = {work.frame_bytes(esz):.0f} B per frame, over the step time"},
            "roofline_smem": smem_roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            **{k: v for k, v in extras.items() if k.startswith("e2e")},
            "f32_context": f32_ctx,
            "gpu_launches": work.launches(args.batch) * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
