"""Output hash of the float64 line pipelines (c1 box, a 1D kernel, a vertical box): bit-identity
checks across library variants (MD_LIB=...)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1212_2245_b200 as md
g = torch.rand((64, 256, 256), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(9)) * 250 + 3
for name, psf in [("box15h", md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15)),
                  ("box21.5v", md.Psf.uniform_box(md.BlurAxis.VERTICAL, 21.5)),
                  ("gen1d", md.Psf.general_1d(np.exp(-0.5 * ((np.arange(13) - 6) / 2.5) ** 2) / np.exp(-0.5 * ((np.arange(13) - 6) / 2.5) ** 2).sum(), md.BlurAxis.HORIZONTAL))]:
    pipe = md.DeblurPipeline((256, 256), psf, md.DeconvParams())
    out = pipe.run_batch(g).cpu().numpy()
    print(name, hashlib.sha1(out.tobytes()).hexdigest()[:12], pipe.plan.describe)
