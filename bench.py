#!/usr/bin/env python
"""Throughput benchmark of the Wiener + RRRL path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c1|c4] [--dtype float32|float64] [--batch B]

One "step" = the whole pipeline (Wiener init + RRRL iterations) over one batch of B
synthetic frames resident in HBM. ``value`` = frames/s over all ranks (weak scaling: B
frames per GPU per step; frames are independent, no collective on the data path), timed
with CUDA events, max over ranks. ``e2e`` = the same metric through the public host-buffer
entry (md_run_host: pinned float64 H2D + run + D2H inside the timed region).
``--impl reference`` times the CPU oracle port of the reference algorithm on all host
cores (one process per core), the CPU baseline arm.

Workloads:
  c1  256x256, uniform horizontal box L=15, Gaussian noise sigma=5, Wiener + 5 RRRL
      (BASELINE.json configs[0], the metric's 256^2 Wiener+RRRL frame).
  c4  256x256 frames with a seeded 1/3 box / 1/3 general-1D / 1/3 2D-line mix (configs[3]);
      each class runs as its own batch through its own plan.
"""

from __future__ import annotations

import argparse
import json
import math
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


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------------------------- inputs

def c1_psf(md):
    return md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15)


def make_frames(md, psf, count: int, distinct: int = 64, sigma: float = 5.0, seed0: int = 5) -> np.ndarray:
    """``count`` float64 frames: the deterministic scene blurred on the GPU (clamped spatial
    convolution), plus ``distinct`` PCG64 noise realisations, quantised, tiled to ``count``."""
    g = md.make_test_image(W, H, seed=7)
    blurred = md.synth_blur(g, psf, quantize_output=True).values
    k = min(distinct, count)
    base = np.empty((k, H, W))
    for i in range(k):
        noisy = blurred + np.random.default_rng(seed0 + i).normal(0.0, sigma, blurred.shape)
        base[i] = np.clip(np.floor(np.clip(noisy, 0.0, 255.0) + 0.5), 0.0, 255.0)
    reps = -(-count // k)
    return np.tile(base, (reps, 1, 1))[:count]


# ---------------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------------- CPU arm

def _cpu_worker(args):
    frames, kind = args
    from oracle import wr3l_oracle as O
    psf = O.make_psf("box", axis="h", length=15)
    params = O.OParams()
    t0 = time.perf_counter()
    for f in frames:
        O.pipeline(f, psf, params, "box")
    return time.perf_counter() - t0


def cpu_rate(frames: np.ndarray, cores: int, per_core: int, pool=None) -> tuple[float, float]:
    """frames/s of the oracle port (reference algorithm, float64) over ``cores`` processes."""
    jobs = [(frames[(i * per_core + np.arange(per_core)) % len(frames)], "c1") for i in range(cores)]
    own = pool is None
    if own:
        pool = mp.get_context("fork").Pool(cores)
    t0 = time.perf_counter()
    pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    if own:
        pool.close()
        pool.join()
    return cores * per_core / wall, wall


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, rank: int) -> None:
    """--impl reference: the reference algorithm (CPU oracle port) on all host cores."""
    if rank != 0:
        return
    cores = host_cores()
    per_core = args.cpu_frames_per_core
    import paper_1212_2245_b200 as md
    frames = make_frames(md, c1_psf(md), 64)
    pool = mp.get_context("fork").Pool(cores)
    for _ in range(args.warmup):
        cpu_rate(frames, cores, per_core, pool)
    rates, walls = [], []
    for _ in range(args.steps):
        r, w = cpu_rate(frames, cores, per_core, pool)
        rates.append(r)
        walls.append(w)
    pool.close()
    pool.join()
    total_frames = cores * per_core * args.steps
    value = total_frames / sum(walls)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(walls) / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic scene, box blur, PCG64 noise)",
        "config": {"workload": "c1: 256x256 box L=15 horizontal, sigma=5, Wiener + 5 RRRL",
                   "frames_per_step": cores * per_core},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": "port",
                         "sample": f"{cores * per_core} frames per step, oracle/wr3l_oracle.pipeline "
                                   f"(NumPy float64, reference radix-2 FFT), one process per core"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "p50_ms_per_frame": 1e3 * statistics.median(walls) / per_core,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------- GPU arm

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1", choices=["c1"])
    ap.add_argument("--dtype", default="float32", choices=["float32", "float64"])
    ap.add_argument("--batch", type=int, default=4096, help="frames per GPU per step")
    ap.add_argument("--e2e-batch", type=int, default=4096)
    ap.add_argument("--cpu-frames-per-core", type=int, default=24)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--fused", default="auto", choices=["auto", "on", "off"])
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1212_2245_b200 as md

    psf = c1_psf(md)
    params = md.DeconvParams()
    fused = None if args.fused == "auto" else args.fused == "on"
    pipe = md.DeblurPipeline((H, W), psf, params, md.Scenario.BOX_1D, dtype=args.dtype, fused=fused)
    plan = pipe.plan
    tdt = torch.float32 if args.dtype == "float32" else torch.float64
    esz = 4 if args.dtype == "float32" else 8
    host = make_frames(md, psf, args.batch)
    f = torch.from_numpy(host).to(device="cuda", dtype=tdt).contiguous()
    u = torch.empty_like(f)
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        plan.run(f, out=u)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    prof = {"init_ms": 0.0, "iter_ms": 0.0, "layout_ms": 0.0, "groups": 0}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            p = plan.run_profile(f, out=u)          # CUDA events between launch groups, same stream
            for k in prof:
                prof[k] += p[k]
        ev1.record(stream)
        torch.cuda.synchronize()
    elapsed_ms = ev0.elapsed_time(ev1)
    t = torch.tensor([elapsed_ms], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    frames_total = args.batch * args.steps * world
    value = frames_total / (max_ms / 1e3)

    # single-frame latency (p50 over 50 runs, batch = 1)
    f1 = f[:1].clone()
    u1 = torch.empty_like(f1)
    lat = []
    for i in range(60):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.run(f1, out=u1)
        b.record(stream)
        b.synchronize()
        if i >= 10:
            lat.append(a.elapsed_time(b))

    # end to end through the public host-buffer entry (DeblurPipeline.run_batch(ndarray) ->
    # md_run_host_ex): pinned host frames in, pinned host results out, copies inside the timed
    # region. Primary: the workload's native 8-bit frames in, float32 results out; also the
    # drop-in float64 -> float64 (reference Image semantics).
    def e2e_rate(in_dtype, out_dtype, nb):
        hin = torch.from_numpy(host[:nb].astype(in_dtype)).pin_memory()
        hout = torch.empty(hin.shape, dtype=torch.from_numpy(np.zeros(1, out_dtype)).dtype).pin_memory()
        hin_np, hout_np = hin.numpy(), hout.numpy()
        pipe.run_batch(hin_np, out=hout_np)
        torch.cuda.synchronize()
        steps = max(3, args.steps // 2)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            pipe.run_batch(hin_np, out=hout_np)   # H2D + convert + run + convert + D2H, synchronous
        el = time.perf_counter() - t0
        te = torch.tensor([el], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        return nb * steps * world / float(te.item()), hin_np.nbytes, hout_np.nbytes

    nb = min(args.e2e_batch, args.batch)
    e2e_value, e2e_in, e2e_out = e2e_rate(np.uint8, np.float32, nb)
    e2e64_value, e2e64_in, e2e64_out = e2e_rate(np.float64, np.float64, min(nb, 1024))

    if rank == 0:
        pk = peaks()
        px = H * W
        iters = params.iterations
        # algorithmic bytes: 8 field passes per RRRL iteration, 2 for Wiener-1D
        iter_bytes_total = 8 * px * esz * args.batch * iters * args.steps
        if plan.fused:
            iter_bytes_total = (2 + 8 * iters) * px * esz * args.batch * args.steps
        achieved = iter_bytes_total / (prof["iter_ms"] / 1e3) / 1e9 if prof["iter_ms"] > 0 else None
        cpu = None
        if not args.no_cpu:
            cores = host_cores()
            r, wall = cpu_rate(host[:64], cores, args.cpu_frames_per_core)
            cpu = {"value": r, "unit": "frames/s", "cores": cores, "kind": "port",
                   "sample": f"{cores * args.cpu_frames_per_core} c1 frames ({wall:.1f} s wall) through "
                             f"oracle/wr3l_oracle.pipeline (NumPy float64), one process per core"}
        step_ms = max_ms / args.steps
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if args.dtype == "float32" else "f64",
            "data": "synthetic (deterministic scene, GPU clamped box blur, PCG64 sigma=5 noise, 8-bit)",
            "config": {"workload": "c1: 256x256 box L=15 horizontal, sigma=5, Wiener + 5 RRRL "
                                   "(BASELINE.json configs[0])",
                       "frames_per_gpu_per_step": args.batch, "parallelism": f"frame-sharded x{world}",
                       "l2": f"inputs {args.batch * px * esz / 2**20:.0f} MiB per GPU > 126 MB L2",
                       "plan": plan.describe},
            "p50_ms_per_frame_batch1": statistics.median(lat),
            "stage_ms_per_step": {k: prof[k] / args.steps for k in ("init_ms", "iter_ms", "layout_ms")},
            "roofline": {"bound": "hbm", "kernel": "RRRL iteration" + (" (fused)" if plan.fused else ""),
                         "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": (achieved / pk["hbm_gbs"]) if achieved else None, "traffic": None,
                         "peak_source": pk["source"],
                         "bytes_model": "SURVEY.md 8(d): 8 field passes per iteration x 65536 px x "
                                        f"{esz} B per frame"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": e2e_in,
                    "d2h_bytes_per_step": e2e_out, "frames_per_step": nb,
                    "entry": "DeblurPipeline.run_batch(pinned uint8 frames) -> float32 results "
                             "(md_run_host_ex, copies pipelined over 3 streams)"},
            "e2e_f64": {"value": e2e64_value, "unit": "frames/s", "h2d_bytes_per_step": e2e64_in,
                        "d2h_bytes_per_step": e2e64_out, "frames_per_step": min(nb, 1024),
                        "entry": "DeblurPipeline.run_batch(pinned float64) -> float64 (drop-in Image semantics)"},
            "gpu_launches": plan.launch_count(args.batch) * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
