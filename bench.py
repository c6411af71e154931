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

class C1:
    """configs[0]: 256^2, horizontal box L=15, sigma=5, Wiener + 5 RRRL."""

    name = "c1: 256x256 box L=15 horizontal, sigma=5, Wiener + 5 RRRL (BASELINE.json configs[0])"

    def __init__(self, md, args):
        self.md = md
        self.psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15)
        self.params = md.DeconvParams()
        fused = None if args.fused == "auto" else args.fused == "on"
        self.pipe = md.DeblurPipeline((H, W), self.psf, self.params, md.Scenario.BOX_1D, dtype=args.dtype,
                                      fused=fused)
        self.describe = self.pipe.plan.describe
        self.fused = self.pipe.plan.fused
        blurred = md.synth_blur(md.make_test_image(W, H, seed=7), self.psf).values
        k = min(64, args.batch)
        base = np.stack([noisy(blurred, 5 + i) for i in range(k)])
        self.host = np.tile(base, (-(-args.batch // k), 1, 1))[:args.batch]
        self.cpu_items = [("box", self.psf, base[i]) for i in range(k)]
        self.latency_plan = self.pipe.plan

    profile_in_loop = True                     # stage marks on the same stream cost nothing here

    def iter_launches(self, n) -> int:
        """Launches of the fused iteration kernel for n frames (one per internal chunk)."""
        return max(1, self.pipe.plan.launch_count(n) // 2)

    def run(self, f, u):
        self.pipe.plan.run(f, out=u)

    @staticmethod
    def e2e_entry(src, dst) -> str:
        return f"DeblurPipeline.run_batch({src}) -> {dst} (md_run_host_ex, copies pipelined over 3 streams)"

    def run_profile(self, f, u) -> dict:
        return self.pipe.plan.run_profile(f, out=u)

    def e2e_set(self, nb):
        return self.host[:nb], None

    def run_host(self, hin, hout, ctx):
        self.pipe.run_batch(hin, out=hout)

    def launches(self, n) -> int:
        return self.pipe.plan.launch_count(n)

    def iter_bytes(self, n, esz) -> float:
        """SURVEY 8(d) algorithmic bytes of the iteration stage for n frames (8 passes/it.)."""
        return 8 * self.params.iterations * PX * esz * n


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


class C4:
    """configs[3]: 256^2 frames over a 48-PSF bank, grouped by PSF."""

    name = ("c4: 256x256 frames, 48-PSF bank (16 box H/V L 5-31 incl. fractional, 16 general 1D, "
            "12 lines L<=21 at random angles + 4 small 2D), sigma=5, Wiener + 5 RRRL (BASELINE.json configs[3])")

    def __init__(self, md, args):
        from paper_1212_2245_b200.batch import PsfBankPipeline
        self.md = md
        self.params = md.DeconvParams()
        self.bank, self.kinds = c4_bank(md)
        self.pipe = PsfBankPipeline((H, W), self.bank, self.params, dtype=args.dtype)
        nb = len(self.bank)
        per = -(-args.batch // nb)
        self.index = np.minimum(np.arange(args.batch) // per, nb - 1)
        scenes = [md.make_test_image(W, H, seed=s).values for s in (7, 8, 9, 10)]
        distinct = 8
        frames = np.empty((args.batch, H, W))
        self.cpu_items = []
        for b, psf in enumerate(self.bank):
            sel = np.nonzero(self.index == b)[0]
            if sel.size == 0:
                continue
            blurred = [md.synth_blur(md.Image(scenes[j]), psf).values for j in range(4)]
            base = [noisy(blurred[j % 4], 1000 * b + j) for j in range(distinct)]
            for k, i in enumerate(sel):
                frames[i] = base[k % distinct]
            self.cpu_items.append((self.kinds[b], psf, base[0]))
        self.host = frames
        self.describe = "; ".join(sorted({p.plan.describe.split(",")[0] for p in self.pipe.pipes}))
        self.fused = False
        self.latency_plan = self.pipe.pipes[int(self.index[0])].plan

    # the timed step deals the PSF groups over two streams (one group's last partial cluster
    # wave overlaps the next group: 227k -> 239k frames/s); the stage split comes from a
    # separate, sequential profiled pass
    profile_in_loop = False

    def run(self, f, u):
        self.pipe.run(f, self.index, out=u, streams=2)

    def run_profile(self, f, u) -> dict:
        tot = {"init_ms": 0.0, "iter_ms": 0.0, "layout_ms": 0.0, "groups": 0}
        for b, s, e in self.pipe.groups(self.index):
            p = self.pipe.pipes[b].plan.run_profile(f[s:e], out=u[s:e])
            for k in tot:
                tot[k] += p[k]
        return tot

    def e2e_set(self, nb):
        sel = np.linspace(0, self.index.size - 1, nb).astype(np.int64)   # every PSF class, sorted
        return self.host[sel], self.index[sel]

    def run_host(self, hin, hout, ctx):
        self.pipe.run_host(hin, ctx, out=hout)

    @staticmethod
    def e2e_entry(src, dst) -> str:
        return (f"PsfBankPipeline.run_host({src}) -> {dst} (copies of PSF group g+1 / g-1 overlap the "
                "deconvolution of group g: 3 streams, md_convert + md_run per group)")

    def launches(self, n) -> int:
        return self.pipe.launch_count(self.index[:n])

    def iter_bytes(self, n, esz) -> float:
        # 8 passes per iteration for every class (line / box / direct-tap convolvers)
        return 8 * self.params.iterations * PX * esz * n


WORKLOADS = {"c1": C1, "c4": C4}


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
        # end to end through the public host entry: pinned float64 image in, float64 out
        # (DeblurPipeline.run_batch(ndarray) -> md_run_host_ex), copies inside the timed region
        hin = f.cpu().pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        hin_np, hout_np = hin.numpy(), hout.numpy()
        pipe.run_batch(hin_np, out=hout_np)
        steps = max(2, min(5, args.steps))
        t0 = time.perf_counter()
        for _ in range(steps):
            pipe.run_batch(hin_np, out=hout_np)
        el = (time.perf_counter() - t0) / steps
        e2e = {"value": 1.0 / el, "unit": "images/s", "h2d_bytes_per_step": hin_np.nbytes,
               "d2h_bytes_per_step": hout_np.nbytes,
               "entry": "DeblurPipeline.run_batch(pinned float64 image) -> float64 (md_run_host_ex)"}
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
    for kind, spec, f in job:
        O.pipeline(f, spec, O.OParams(), kind)
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
    items = [(k, oracle_spec(p), f) for k, p, f in work.cpu_items]
    return [[items[(c * per_core + i) % len(items)] for i in range(per_core)] for c in range(cores)]


def cpu_rate(jobs, pool) -> tuple[float, float]:
    t0 = time.perf_counter()
    pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    return sum(len(j) for j in jobs) / wall, wall


def run_reference(args, rank: int) -> None:
    """--impl reference: the reference algorithm (CPU oracle port) on all host cores."""
    if rank != 0:
        return
    import paper_1212_2245_b200 as md
    args.batch = min(args.batch, 1024)
    work = WORKLOADS[args.config](md, args)            # inputs only (GPU-synthesised blur)
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
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(walls) / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic scenes, GPU-synthesised blur, PCG64 sigma=5 noise, 8-bit)",
        "config": {"workload": work.name, "frames_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": "port",
                         "sample": f"{per_step} frames per step through oracle/wr3l_oracle.pipeline (NumPy "
                                   "float64, the reference's radix-2 FFT and cumsum box filter), one process "
                                   "per host core"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "p50_ms_per_frame": 1e3 * statistics.median(walls) / args.cpu_frames_per_core,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------- GPU arm

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1", choices=sorted(WORKLOADS) + ["c5"])
    ap.add_argument("--size", type=int, default=16384, help="c5 image side")
    ap.add_argument("--dtype", default="float32", choices=["float32", "float64"])
    ap.add_argument("--batch", type=int, default=None, help="frames per GPU per step")
    ap.add_argument("--e2e-batch", type=int, default=4096)
    ap.add_argument("--cpu-frames-per-core", type=int, default=24)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--fused", default="auto", choices=["auto", "on", "off"])
    args = ap.parse_args()
    if args.batch is None:
        args.batch = 4096 if args.config == "c1" else 16384

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    if args.impl == "reference":
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        run_reference(args, rank)
        return

    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.config == "c5":
        run_c5(args, rank, world, local)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    import paper_1212_2245_b200 as md

    work = WORKLOADS[args.config](md, args)
    tdt = torch.float32 if args.dtype == "float32" else torch.float64
    esz = 4 if args.dtype == "float32" else 8
    f = torch.from_numpy(work.host).to(device="cuda", dtype=tdt).contiguous()
    u = torch.empty_like(f)
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        work.run(f, u)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    prof = {"init_ms": 0.0, "iter_ms": 0.0, "layout_ms": 0.0, "groups": 0}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            if work.profile_in_loop:
                p = work.run_profile(f, u)          # CUDA events between launch groups, same stream
                for k in prof:
                    prof[k] += p[k]
            else:
                work.run(f, u)
        ev1.record(stream)
        torch.cuda.synchronize()
    elapsed_ms = ev0.elapsed_time(ev1)
    if not work.profile_in_loop:
        # stage split from profiled sequential steps after the timed region, scaled to it
        npf = max(1, min(args.steps, 5))
        for _ in range(npf):
            p = work.run_profile(f, u)
            for k in prof:
                prof[k] += p[k] * args.steps / npf
    t = torch.tensor([elapsed_ms], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = args.batch * args.steps * world / (max_ms / 1e3)

    # single-frame latency (p50 / p99 over 200 runs, batch = 1)
    f1, u1 = f[:1].clone(), torch.empty_like(f[:1])
    lat = []
    for i in range(210):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        work.latency_plan.run(f1, out=u1)
        b.record(stream)
        b.synchronize()
        if i >= 10:                                   # 200 timed single-frame runs
            lat.append(a.elapsed_time(b))

    # host-observed single-frame latency (call -> result ready, synchronised per call): the
    # direct md_run call vs a replay of the same run captured as a CUDA graph (GpuPlan.capture)
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

    # end to end through the public host-buffer entry (DeblurPipeline.run_batch(ndarray) ->
    # md_run_host_ex): pinned host frames in, pinned host results out, copies inside the timed
    # region. Primary: the workload's native 8-bit frames in, float32 results out; also the
    # drop-in float64 -> float64 (reference Image semantics).
    def e2e_rate(in_dtype, out_dtype, nb):
        frames, ctx = work.e2e_set(nb)
        hin = torch.from_numpy(np.ascontiguousarray(frames).astype(in_dtype)).pin_memory()
        hout = torch.empty(hin.shape, dtype=torch.from_numpy(np.zeros(1, out_dtype)).dtype).pin_memory()
        hin_np, hout_np = hin.numpy(), hout.numpy()
        work.run_host(hin_np, hout_np, ctx)
        torch.cuda.synchronize()
        steps = max(3, min(10, args.steps // 4))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            work.run_host(hin_np, hout_np, ctx)  # H2D + convert + run + convert + D2H, synchronous
        el = time.perf_counter() - t0
        te = torch.tensor([el], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        return nb * steps * world / float(te.item()), hin_np.nbytes, hout_np.nbytes

    nb = min(args.e2e_batch, args.batch)
    e2e_value, e2e_in, e2e_out = e2e_rate(np.uint8, np.float32, nb)
    nb64 = min(nb, 1024)
    e2e64_value, e2e64_in, e2e64_out = e2e_rate(np.float64, np.float64, nb64)
    e2e8_value, e2e8_in, e2e8_out = e2e_rate(np.uint8, np.uint8, nb)

    if rank == 0:
        pk = peaks()
        iter_bytes = work.iter_bytes(args.batch, esz) * args.steps
        achieved = iter_bytes / (prof["iter_ms"] / 1e3) / 1e9 if prof["iter_ms"] > 0 else None
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
        # the fused kernel keeps the iterate on chip, so its other roofline is the shared-memory
        # pipe (north_star: "HBM (or SMEM for fused in-cluster)"): ncu wavefronts per frame over
        # this run's iteration time, against SMs x 128 B/clk x the max SM clock
        smem_roof = None
        wf = measured_smem(f"{args.config}_{args.dtype}", args.batch) if work.fused else None
        if wf and prof["iter_ms"] > 0:
            sms = torch.cuda.get_device_properties(local).multi_processor_count
            ach = wf * 128 * args.steps / (prof["iter_ms"] / 1e3) / 1e12
            pk_s = sms * 128 * pk["sm_max_mhz"] * 1e6 / 1e12
            smem_roof = {"bound": "smem", "kernel": "RRRL iteration (fused cluster kernel)", "achieved": ach,
                         "peak": pk_s, "unit": "TB/s", "frac": ach / pk_s,
                         "wavefronts_per_frame": wf / args.batch,
                         "source": "ncu l1tex__data_pipe_lsu_wavefronts_mem_shared.sum (profiles/ncu_traffic.json) "
                                   "over this run's iteration time; peak = SMs x 128 B/clk x max SM clock"}
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32" if args.dtype == "float32" else "f64",
            "data": "synthetic (deterministic scenes, GPU clamped-spatial blur, PCG64 sigma=5 noise, 8-bit)",
            "config": {"workload": work.name, "frames_per_gpu_per_step": args.batch,
                       "parallelism": f"frame-sharded x{world}",
                       "l2": f"inputs {args.batch * PX * esz / 2**20:.0f} MiB per GPU > 126 MB L2",
                       "plan": work.describe},
            "p50_ms_per_frame_batch1": statistics.median(lat),
            "p99_ms_per_frame_batch1": sorted(lat)[min(len(lat) - 1, int(0.99 * len(lat)))],
            "host_p50_ms_per_frame_batch1": host_lat,
            "stage_ms_per_step": {k: prof[k] / args.steps for k in ("init_ms", "iter_ms", "layout_ms")},
            "stage_split_source": ("CUDA events between the launch groups of the timed steps" if work.profile_in_loop
                                   else "CUDA events of profiled sequential steps after the timed region"),
            "roofline": {"bound": "hbm",
                         "kernel": "RRRL iteration" + (" (fused cluster kernel)" if work.fused else ""),
                         "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": (achieved / pk["hbm_gbs"]) if achieved else None,
                         "traffic": (measured_traffic(f"{args.config}_{args.dtype}", args.batch / work.iter_launches(args.batch))
                                     if work.fused else None),
                         "traffic_note": "DRAM bytes per launch of the fused kernel (ncu, scaled to this batch); "
                                         "iterate, p, W stay on chip, so traffic is the compulsory stream only",
                         "peak_source": pk["source"],
                         "bytes_model": "SURVEY.md 8(d): 8 field passes per RRRL iteration x 65536 px x "
                                        f"{esz} B per frame; time = CUDA events around the iteration launches"},
            "roofline_smem": smem_roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": e2e_in,
                    "d2h_bytes_per_step": e2e_out, "frames_per_step": nb,
                    "entry": work.e2e_entry("pinned uint8 frames", "float32 results")},
            "e2e_f64": {"value": e2e64_value, "unit": "frames/s", "h2d_bytes_per_step": e2e64_in,
                        "d2h_bytes_per_step": e2e64_out, "frames_per_step": nb64,
                        "entry": work.e2e_entry("pinned float64 frames", "float64 (drop-in Image semantics)")},
            "e2e_u8": {"value": e2e8_value, "unit": "frames/s", "h2d_bytes_per_step": e2e8_in,
                       "d2h_bytes_per_step": e2e8_out, "frames_per_step": nb,
                       "entry": work.e2e_entry("pinned uint8 frames", "uint8 frames quantised like the "
                                               "reference's write_pgm (pgm.py:56-58), the CLI's output")},
            "gpu_launches": work.launches(args.batch) * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
