"""c4 bank: PsfBankPipeline.run with the PSF groups on 1 / 2 / 3 / 4 streams (bench c4 frames)."""
import os, sys, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1212_2245_b200 as md
from bench import C4

work = C4(md, types.SimpleNamespace(dtype="float32", batch=16384))
f = work.device_frames(torch.float32)
u = torch.empty_like(f)
ref = None
for ns in (1, 2, 3, 4, 1):
    for _ in range(2):
        work.pipe.run(f, work.index, out=u, streams=ns)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        work.pipe.run(f, work.index, out=u, streams=ns)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 5
    if ref is None:
        ref = u.clone()
    same = bool(torch.equal(ref, u))
    print(f"streams={ns}: {ms:.2f} ms per 16384 frames = {16384 / ms * 1e3:.0f} frames/s, bitwise equal {same}", flush=True)
