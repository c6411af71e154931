"""Horizontal vs vertical box lines (1024 frames, float64): for ncu captures of the line Wiener (the vertical one transposes)."""
import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, paper_1212_2245_b200 as md
g = torch.rand((1024, 256, 256), dtype=torch.float64, device="cuda") * 250 + 3
for ax in (md.BlurAxis.HORIZONTAL, md.BlurAxis.VERTICAL):
    pipe = md.DeblurPipeline((256, 256), md.Psf.uniform_box(ax, 15), md.DeconvParams())
    u = torch.empty_like(g)
    pipe.plan.run(g, out=u); torch.cuda.synchronize()
