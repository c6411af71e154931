"""Generate tests/golden/big_c5_4096.npz by running the REFERENCE package itself on the c5
workload at 4096^2 (build container only; about 4 minutes of CPU).

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_c5.py

SURVEY.md 8(d) c5: line PSF L=21 at 30 deg (Psf.line rasteriser -> general_2d), noise-free,
default DeconvParams (5 iterations), Scenario.FOURIER_2D (deconv.py:653-690), the scene from
the reference's make_test_image and its synth_blur (synth.py:34-41, 90-126). The full 128 MB
result is not committed; the fixture keeps what a size-independent parity check needs:
  * sha256 of the input frame (the GPU box regenerates it and must get the same bytes);
  * every row within 2 rows of each 8-slab boundary (rows 512 k - 2 .. 512 k + 1, wrapping),
    where a row-slab decomposition would go wrong first;
  * 20,000 seeded random pixels, the per-row and per-column means;
  * the PSNR of the result against the sharp scene, and the reference's wall time.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "big_c5_4096.npz")
N = 4096
SLABS = 8


def boundary_rows(n: int = N, slabs: int = SLABS) -> np.ndarray:
    rows = set()
    for k in range(slabs):
        for d in (-2, -1, 0, 1):
            rows.add((k * (n // slabs) + d) % n)
    return np.array(sorted(rows), dtype=np.int64)


def sample_pixels(n: int = N, count: int = 20000) -> tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng(4096)
    return rng.integers(0, n, count), rng.integers(0, n, count)


def main() -> None:
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, os.path.dirname(HERE))
    import motiondeblur as md
    from motiondeblur.core import Psf
    from motiondeblur.deconv import DeblurPipeline, Scenario
    from paper_1212_2245_b200.core import Psf as LinePsf   # rasteriser only (host numpy)

    line = LinePsf.line(21.0, 30.0)
    psf = Psf.general_2d(np.asarray(line.weights), center=tuple(int(c) for c in line.center))
    g = md.make_test_image(N, N, seed=7)
    f = md.synth_blur(g, psf)
    params = md.DeconvParams()
    t0 = time.perf_counter()
    u = DeblurPipeline(f.shape, psf, params, Scenario.FOURIER_2D).run(f).values
    wall = time.perf_counter() - t0
    psnr = 10.0 * np.log10(255.0 ** 2 / np.mean((u - g.values) ** 2))
    rows = boundary_rows()
    py, px = sample_pixels()
    np.savez_compressed(
        OUT, f_sha256=np.array(hashlib.sha256(np.ascontiguousarray(f.values).tobytes()).hexdigest()),
        rows=rows, row_values=u[rows], py=py, px=px, pix_values=u[py, px],
        row_means=u.mean(axis=1), col_means=u.mean(axis=0), psnr=np.array(psnr),
        ref_wall_s=np.array(wall), psf_weights=np.asarray(line.weights), psf_center=np.asarray(line.center),
        params=np.array([params.wiener_k, params.alpha, params.iterations, params.eps_data, params.eps_reg,
                         params.floor]))
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes); reference run {wall:.1f} s, PSNR {psnr:.4f} dB")


if __name__ == "__main__":
    main()
