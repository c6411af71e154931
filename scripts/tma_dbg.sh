for m in 1 2 3; do echo "mask $m"; MD_PLANE_TMA_MASK=$m CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/c4_2d_probe.py 64 2>&1 | tail -2; done
for m in 1 2; do echo "f32 mask $m"; MD_PLANE_TMA_MASK=$m CUDA_LAUNCH_BLOCKING=1 timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_1212_2245_b200 as md
psf = md.Psf.line(15.0, 40.0)
for n in (64, 128, 256, 512):
  for dt in ('float64','float32'):
    g = torch.rand((3, n, n), dtype=torch.float64, device='cuda') * 255
    p = md.DeblurPipeline((n, n), psf, md.DeconvParams(), md.Scenario.FOURIER_2D, dtype=dt, fused=False)
    try:
        p.run_batch(g if dt=='float64' else g.float()); torch.cuda.synchronize(); print(n, dt, 'ok', p.plan.describe)
    except Exception as e:
        print(n, dt, 'FAIL', str(e)[:80]); break
" 2>&1 | tail -9; done
