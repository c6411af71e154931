"""c1 chunk pipeline probe (bench c1 frames): Wiener-only, one chunk, and pipelined chunk sizes."""
import os, sys, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1212_2245_b200 as md
from bench import C1

args = types.SimpleNamespace(fused="auto", dtype="float32", batch=4096)
work = C1(md, args)
f = torch.from_numpy(work.host).cuda().float()
u = torch.empty_like(f)


def timed(plan, f, u, reps=10):
    for _ in range(3):
        plan.run(f, out=u)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        plan.run(f, out=u)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


w0 = md.DeblurPipeline((256, 256), work.psf, md.DeconvParams(iterations=0), dtype="float32").plan
p5 = work.pipe.plan
for n in (33, 330, 1056, 1365, 4096):
    p5.set_chunk(n)
    tw, t1 = timed(w0, f[:n], u[:n]), timed(p5, f[:n], u[:n])
    print(f"one chunk of {n}: W {tw:.3f} ms, W+F {t1:.3f} ms -> F {1e3 * (t1 - tw) / n:.3f} us/frame", flush=True)
for n in (1056, 1365, 2048, 4096):
    p5.set_chunk(n)
    t = timed(p5, f, u)
    print(f"4096 frames in chunks of {n}: {t:.3f} ms = {4096 / t * 1e3:.0f} frames/s", flush=True)
p5.set_chunk(0)
print("auto:", round(timed(p5, f, u), 3), "ms")
