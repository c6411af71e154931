"""Two-level-FFT Wiener (big_fft plans, the c5 route): output hash and init time per library
variant (MD_LIB=...), for bit-identity checks of FFT-pass changes.

    python scripts/wiener_hash_probe.py [sizes...]      (default 4096 16384)"""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1212_2245_b200 as md

sizes = [int(x) for x in sys.argv[1:]] or [4096, 16384]
psf = md.Psf.line(21.0, 30.0)
for n in sizes:
    g = torch.rand((1, n, n), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5)) * 250 + 3
    pipe = md.DeblurPipeline((n, n), psf, md.DeconvParams(iterations=0), big_fft=True)
    u = torch.empty_like(g)
    pipe.plan.run(g, out=u)
    h = hashlib.sha1(u.cpu().numpy().tobytes()).hexdigest()[:12]
    ts = sorted(pipe.plan.run_profile(g, out=u)["init_ms"] for _ in range(5))
    print(f"n={n} hash={h} wiener_ms={ts[len(ts) // 2]:.3f} (min {ts[0]:.3f})", flush=True)
    del g, u, pipe
    torch.cuda.empty_cache()
