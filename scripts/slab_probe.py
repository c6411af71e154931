"""Bisect helper: run_slabs(n, world) vs the single plan for one configuration (own process)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1212_2245_b200 as md
from paper_1212_2245_b200.slab import run_slabs

n, world, its = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 1
mode = sys.argv[4] if len(sys.argv) > 4 else "both"
psf = md.Psf.line(21.0, 30.0)
f = torch.rand((n, n), device="cuda", dtype=torch.float64) * 200 + 20
pipe = md.DeblurPipeline((n, n), psf, md.DeconvParams(iterations=its), big_fft=True)
if mode in ("both", "single"):
    want = pipe.run_batch(f)
    torch.cuda.synchronize()
    print("single ok", flush=True)
if mode in ("both", "slabs"):
    got = run_slabs(pipe.plan, f, world)
    torch.cuda.synchronize()
    print("slabs ok", flush=True)
if mode == "both":
    print(n, world, its, "max|d|", float((got - want).abs().max()), flush=True)
