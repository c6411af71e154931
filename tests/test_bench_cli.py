"""bench.py's own logic on CPU: the frame-sharded timing path under `--gpus 2` (ranks
self-launched, gloo process group, barrier + max over ranks), and the reference arm, which
must run the CPU oracle without touching the device or loading libmdcuda.so."""

from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, extra_env=None, timeout=300):
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1", **(extra_env or {}))
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, *args], cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_gpus2_self_launch_gloo():
    d = _run(["bench.py", "--gpus", "2", "--backend", "gloo", "--steps", "3", "--warmup", "1", "--batch", "16"])
    assert d["n_gpus"] == 2 and d["steps"] == 3
    assert d["config"]["parallelism"] == "frame-sharded x2"
    assert d["config"]["frames_per_gpu_per_step"] == 16
    assert d["value"] > 0


def test_reference_arm_is_device_free():
    probe = (
        "import runpy, sys\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', "
        "'--cpu-frames-per-core', '1', '--batch', '64']\n"
        "try:\n"
        "    runpy.run_path('bench.py', run_name='__main__')\n"
        "finally:\n"
        "    maps = open('/proc/self/maps').read()\n"
        "    sys.stderr.write('LIBMDCUDA_MAPPED=%d\\n' % ('libmdcuda' in maps))\n"
    )
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1", CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "-c", probe], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "LIBMDCUDA_MAPPED=0" in r.stderr
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["impl"] == "reference" and d["dtype"] == "f64"
    # the same config object the GPU arm prints for the same command line
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.bench_config(bench.C1.name, 64, 1, 8)
    assert d["cpu_baseline"]["kind"] == "port" and d["e2e"]["h2d_bytes_per_step"] == 0


def test_c4_strong_scaling_split():
    """configs[3]: one global batch dealt round-robin over the ranks (every rank gets every PSF
    class, the per-rank batches sum to the global one)."""
    sys.path.insert(0, ROOT)
    import bench
    import numpy as np
    import paper_1212_2245_b200 as md
    parts = []
    for r in range(4):
        os.environ.update({"WORLD_SIZE": "4", "RANK": str(r)})
        try:
            a = bench.parse_args(["--config", "c4", "--global-batch", "480"])
        finally:
            os.environ.pop("WORLD_SIZE"), os.environ.pop("RANK")
        assert a.batch == 120 and a.scaling == "strong" and a.world == 4
        w = bench.C4(md, a, bench.cpu_synth(md), gpu=False)
        assert np.all(np.diff(w.index) >= 0) and set(w.index.tolist()) == set(range(48))
        parts.append(w.src)
        cfg = bench.bench_config(w.name, a.batch, a.world, 8, a.global_batch)
        assert cfg["global_batch"] == 480 and cfg["frames_per_gpu_per_step"] == 120
    whole = np.sort(np.concatenate(parts))
    a1 = bench.parse_args(["--config", "c4", "--global-batch", "480"])
    assert a1.batch == 480 and a1.world == 1
    assert np.array_equal(whole, np.sort(bench.C4(md, a1, bench.cpu_synth(md), gpu=False).src))
    d = bench.parse_args(["--config", "c4"])
    assert d.global_batch == 65536 and d.batch == 65536
    assert bench.parse_args(["--config", "c4", "--batch", "64"]).scaling == "weak"


def test_c2_c3_workloads_host_side():
    """configs[1] / configs[2] bench lines: batch defaults, the SURVEY 8(d) bytes model, CPU
    sample sizing, and the device-free frames the reference arm uses."""
    sys.path.insert(0, ROOT)
    import bench
    import paper_1212_2245_b200 as md
    a2 = bench.parse_args(["--config", "c2"])
    assert a2.batch == 256 and a2.cpu_frames_per_core == 2 and a2.scaling == "weak"
    w2 = bench.C2(md, a2, bench.cpu_synth(md), gpu=False)
    assert w2.frame_bytes(8) == 182452224 and w2.params.iterations == 10
    assert w2.base.shape == (4, 512, 512) and w2.src.size == 256
    a3 = bench.parse_args(["--config", "c3", "--batch", "8"])
    assert a3.batch == 8 and a3.cpu_frames_per_core == 1
    assert bench.C3.passes_per_iteration == 18 and (7 + 18 * 5) * 1024 ** 2 * 8 == 813694976
    assert bench.parse_args(["--config", "c1"]).cpu_frames_per_core == 24
