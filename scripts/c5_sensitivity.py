"""Conditioning of the c5 workload itself (CPU, the oracle = the reference's arithmetic):
run the 4096^2 c5 pipeline (line L=21@30deg, noise-free, 5 RRRL iterations, FOURIER_2D) twice,
the second time with the Wiener start perturbed by 1e-13 relative noise, and report how far
the results drift; also the oracle against the reference's own run (tests/golden/big_c5_4096.npz).
About 4 minutes of CPU. Output recorded in profiles/r2_c5_sensitivity.txt."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import wr3l_oracle as O
import paper_1212_2245_b200 as md
d = np.load(os.path.join(ROOT, 'tests/golden/big_c5_4096.npz'))
g = md.make_test_image(4096, 4096, seed=7).values
spec = O.OPsf("2d", d["psf_weights"], tuple(int(c) for c in d["psf_center"]))
f = np.clip(np.floor(O.clamped_convolve(g, spec) + 0.5), 0, 255)
p = O.OParams()
# pipeline with a perturbed Wiener start: relative 1e-13 noise on u0
hspec = O.spectrum_2d(spec, f.shape)
wien = O.fft2(O.fft2(f) * O.wiener_multiplier(hspec, p.wiener_k), inverse=True).real
conv = O.Fourier2DConv(hspec)
fpos = np.maximum(f, p.floor)
res = []
for eps in (0.0, 1e-13):
    u = np.maximum(wien * (1 + eps * np.random.default_rng(1).standard_normal(wien.shape)), p.floor)
    for _ in range(p.iterations):
        u = O.rrrl_iteration(u, fpos, conv, p)
    res.append(u)
dd = np.abs(res[0] - res[1])
print("max", dd.max(), "at", np.unravel_index(dd.argmax(), dd.shape), ">0.0255:", int((dd > 0.0255).sum()), ">1e-6:", int((dd > 1e-6).sum()))
er = np.abs(res[0][d["rows"]] - d["row_values"])
print("oracle vs reference rows max", er.max())
