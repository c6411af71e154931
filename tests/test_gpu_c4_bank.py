"""configs[3] (c4) parity on the bench's OWN workload: a seeded 256-frame sample of bench.py's
48-PSF bank (16 boxes incl. even / fractional lengths and both axes, 16 general 1D kernels,
12 lines at random angles, 4 small dense 2D kernels; sigma = 5 noise), deblurred in FLOAT32
through PsfBankPipeline exactly as the c4 bench line runs it, against the CPU oracle (float64,
the reference's algorithm) frame by frame. Bar (north_star): max|d| <= 1e-4 * 255 and
|dPSNR| <= 0.01 dB against the sharp scene; every PSF class, the 2D class included."""

from __future__ import annotations

import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4 * 255.0
SAMPLE = 256


def test_c4_bank_sample_float32_vs_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import multiprocessing as mp

    import bench
    import paper_1212_2245_b200 as md
    from paper_1212_2245_b200.batch import PsfBankPipeline
    bank, kinds = bench.c4_bank(md)
    rng = np.random.default_rng(256)
    index = np.sort(np.concatenate([np.arange(len(bank)), rng.integers(0, len(bank), SAMPLE - len(bank))]))
    frames, _, scene_of = bench.c4_frames(md, bank, index, bench.gpu_synth(md), with_scenes=True)
    pipe = PsfBankPipeline((bench.H, bench.W), bank, md.DeconvParams(), dtype="float32")
    got = pipe.run(torch.from_numpy(frames).to("cuda", torch.float32), index).double().cpu().numpy()
    from oracle import wr3l_oracle as O
    specs = [bench.oracle_spec(bank[index[i]]) for i in range(SAMPLE)]
    workers = max(1, min(16, len(os.sched_getaffinity(0))))
    with ProcessPoolExecutor(workers, mp_context=mp.get_context("spawn")) as ex:
        ref = np.stack(list(ex.map(O.pipeline, list(frames), specs, [O.OParams()] * SAMPLE,
                                   [kinds[index[i]] for i in range(SAMPLE)], chunksize=4)))
    scenes = [md.make_test_image(bench.W, bench.H, seed=s).values for s in bench.C4_SCENE_SEEDS]
    worst = {}
    for i in range(SAMPLE):
        err = float(np.abs(got[i] - ref[i]).max())
        g = scenes[scene_of[i]]
        dpsnr = abs(md.psnr(md.Image(got[i]), md.Image(g)) - md.psnr(md.Image(ref[i]), md.Image(g)))
        k = kinds[index[i]]
        worst[k] = max(worst.get(k, (0.0, 0.0)), (err, dpsnr))
        assert err <= TOL, (i, int(index[i]), k, err)
        assert dpsnr <= 0.01, (i, int(index[i]), k, dpsnr)
    assert set(worst) == {"box", "fourier1d", "fourier2d"}
    print("worst (max|d|, dPSNR) per class:", worst)
