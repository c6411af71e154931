"""A/B probe for the two-level FFT passes: output hashes (bit-identity across library variants,
select one with MD_LIB=...) and device time of the large-image Wiener.

python scripts/fft_ab_probe.py            -> one line per case: name, sha1 of the result, ms
"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1212_2245_b200 as md


def sha(t) -> str:
    a = t.detach().cpu().numpy() if torch.is_tensor(t) else np.asarray(t)
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()[:12]


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return (out, float(np.median(ts))) if ts else (fn(), 0.0)


# FFT_AB_PROFILE=1: only the 16384^2 Wiener, run once (for an ncu capture of its passes)
PROFILE = os.environ.get("FFT_AB_PROFILE") == "1"
# 1D transforms through the public FourierPlan (lengths 2^12 .. 2^20: sub-lengths 2^6 .. 2^10)
rng = np.random.default_rng(3)
for lg in (() if PROFILE else (12, 14, 16, 18, 20)):
    n = 1 << lg
    x = torch.from_numpy(rng.standard_normal((4, n)) + 1j * rng.standard_normal((4, n))).cuda()
    plan = md.plan_fft(n)
    y = plan.forward(x.T.contiguous())
    z = plan.inverse(y)
    print(f"fft1d n=2^{lg}", sha(y), sha(z), flush=True)

# the large-image Wiener (two-level passes incl. the fused filter pass)
for n in ((16384,) if PROFILE else (4096, 16384)):
    psf = md.Psf.line(21.0, 30.0)
    g = torch.rand((n, n), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5)) * 255
    pipe = md.DeblurPipeline((n, n), psf, md.DeconvParams(iterations=0))
    out, ms = timed(lambda: pipe.run_batch(g), reps=0 if PROFILE else 5)
    print(f"wiener {n}", sha(out), f"{ms:.3f} ms", pipe.plan.describe, flush=True)
