"""Does work beside the float64 cluster kernel land on the SMs it leaves idle? Time c1 (4096
frames) alone, then with a 28-CTA 100 KB filler on a low-priority stream launched right after."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1212_2245_b200 as md
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsmfiller.so"))
psf = md.Psf.uniform_box(md.BlurAxis.HORIZONTAL, 15)
pipe = md.DeblurPipeline((256, 256), psf, md.DeconvParams(), md.Scenario.BOX_1D)
f = torch.rand((4096, 256, 256), dtype=torch.float64, device="cuda") * 200 + 20
u = torch.empty_like(f)
hi = torch.cuda.Stream(priority=-1)
lo = torch.cuda.Stream(priority=0)
smid = torch.zeros(64, dtype=torch.int32, device="cuda")
for _ in range(2):
    pipe.plan.run(f, out=u, stream=hi)
torch.cuda.synchronize()
def timed(filler):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(hi)
    pipe.plan.run(f, out=u, stream=hi)
    if filler:
        lib.launch_filler(ctypes.c_void_p(lo.cuda_stream), filler, 100 * 1024, ctypes.c_longlong(15_000_000), ctypes.c_void_p(smid.data_ptr()))
    e1.record(hi)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)
for n in (0, 28, 0, 28, 40):
    ms = timed(n)
    print(f"filler CTAs {n:2d}: cluster path {ms:.2f} ms", flush=True)
print("filler SMs:", sorted(set(smid.cpu().numpy()[:40].tolist())))
