"""The c5 row-slab path as REAL processes: world 2 and 4 ranks, each its own process with the
CUDA slab backend (md_slab_* kernels) on the one GPU of this box, exchanging halos and the
Wiener spectrum blocks through a torch.distributed process group (gloo over host-staged copies,
HostStagedComm -- NCCL would move device memory directly on 8 GPUs, where each rank has its own
device). The assembled image must equal the single-plan run (1e-9)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 1024


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(md):
    psf = md.Psf.line(21.0, 30.0)
    f = md.synth_blur(md.make_test_image(N, N, seed=3), psf).values
    return psf, f


def _rank_main(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1212_2245_b200 as md
        from paper_1212_2245_b200.slab import CudaSlabBackend, DistComm, HostStagedComm, SlabGeometry, SlabWorker
        torch.cuda.set_device(0)
        psf, f = _problem(md)
        pipe = md.DeblurPipeline((N, N), psf, md.DeconvParams(iterations=3), big_fft=True)
        be = CudaSlabBackend(pipe.plan)
        geo = SlabGeometry(N, N, rank, world, *be.halo_rows())
        worker = SlabWorker(be, geo, 3, torch.device("cuda", 0), torch.float64)
        S = N // world
        own = torch.from_numpy(f[rank * S:(rank + 1) * S].copy()).cuda()
        res = worker.run(HostStagedComm(DistComm()), own)
        torch.cuda.synchronize()
        np.save(os.path.join(out_dir, f"slab{rank}.npy"), res.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_process_ranks_equal_single_plan(tmp_path, world):
    import torch
    import torch.multiprocessing as tmp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1212_2245_b200 as md
    tmp.spawn(_rank_main, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"slab{r}.npy") for r in range(world)])
    psf, f = _problem(md)
    pipe = md.DeblurPipeline((N, N), psf, md.DeconvParams(iterations=3), big_fft=True)
    want = pipe.run(md.Image(f)).values
    assert np.abs(got - want).max() <= 1e-9
