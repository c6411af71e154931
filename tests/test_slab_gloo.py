"""Row-slab decomposition logic (BASELINE.json configs[4]) on CPU: world_size 2 and 4 over a
gloo process group (DistComm), and 4 thread-ranks (LocalComm), with the NumPy stand-in backend
(tests/slab_numpy_backend.py). The assembled result must equal the oracle's whole-image
Wiener + RRRL pipeline (FOURIER_2D semantics: periodic convolution, Neumann TV)."""

from __future__ import annotations

import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from oracle import wr3l_oracle as O

H = W = 64
ITERS = 3


def _problem():
    rng = np.random.default_rng(77)
    w = np.zeros((7, 9))
    w[3, 1:8] = 1.0
    w[2, 5:8] = 0.5
    w[4, 1:3] = 0.25
    w /= w.sum()
    center = (3, 4)
    f = np.clip(rng.uniform(20, 230, (H, W)), 0, 255).round()
    return w, center, f, O.OParams(iterations=ITERS)


def _reference():
    w, c, f, p = _problem()
    return O.pipeline(f, O.OPsf("2d", w, c), p, "fourier2d")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1212_2245_b200.slab import DistComm, SlabGeometry, SlabWorker
        from slab_numpy_backend import NumpySlabBackend
        w, c, f, p = _problem()
        be = NumpySlabBackend(w, c, p, H, W)
        top, bot = be.halo_rows()
        geo = SlabGeometry(H, W, rank, world, top, bot)
        worker = SlabWorker(be, geo, p.iterations, "cpu", torch.float64)
        S = H // world
        res = worker.run(DistComm(), torch.from_numpy(f[rank * S:(rank + 1) * S].copy()))
        np.save(os.path.join(out_dir, f"slab{rank}.npy"), res.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_slabs_match_whole_image_oracle(tmp_path, world):
    port = _free_port()
    tmp.spawn(_rank_main, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"slab{r}.npy") for r in range(world)])
    np.testing.assert_allclose(got, _reference(), rtol=0, atol=1e-9)


def test_local_thread_ranks_match_oracle():
    from paper_1212_2245_b200.slab import LocalComm, SlabGeometry, SlabWorker
    from slab_numpy_backend import NumpySlabBackend
    world = 4
    w, c, f, p = _problem()
    comm = LocalComm(world)
    S = H // world
    out = [None] * world

    def body(r):
        be = NumpySlabBackend(w, c, p, H, W)
        geo = SlabGeometry(H, W, r, world, *be.halo_rows())
        out[r] = SlabWorker(be, geo, p.iterations, "cpu", torch.float64).run(
            comm, torch.from_numpy(f[r * S:(r + 1) * S].copy())).numpy().copy()

    threads = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    np.testing.assert_allclose(np.concatenate(out), _reference(), rtol=0, atol=1e-9)


def test_geometry_validation():
    from paper_1212_2245_b200.slab import SlabGeometry
    with pytest.raises(ValueError):
        SlabGeometry(64, 64, 0, 3, 2, 2)          # does not divide
    with pytest.raises(ValueError):
        SlabGeometry(64, 64, 0, 32, 4, 4)         # halo deeper than a 2-row slab
    g = SlabGeometry(64, 64, 1, 4, 3, 5)
    assert (g.S, g.Wb, g.row0, g.ext_rows) == (16, 16, 16, 24)
