"""One PSF group of each c4 class (box H/V small and large radius, general 1D H/V, 2D line,
2D dense), the bench's frames: a short command to scan every kernel of the bank under ncu."""
import os, sys, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1212_2245_b200 as md
from bench import C4

work = C4(md, types.SimpleNamespace(dtype="float32", batch=16384))
f_all = work.device_frames(torch.float32)
groups = work.pipe.groups(work.index)
pick = [0, 1, 2, 11, 16, 17, 20, 32, 44]          # box H R14, V R4, H R2, V R14, 1D H, 1D V, 1D H long, 2D line, 2D 7x7
for b, s, e in groups:
    if b not in pick:
        continue
    plan = work.pipe.pipes[b].plan
    f = f_all[s:e]
    u = torch.empty_like(f)
    plan.run(f, out=u)
torch.cuda.synchronize()
print("ok")
