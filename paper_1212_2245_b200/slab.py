"""One large image split into row slabs over ranks (BASELINE.json configs[4], "c5").

SPMD driver: every rank owns ``S = H / world`` consecutive rows plus halo rows and runs

  Wiener:  rows FFT (local) -> all-to-all (row slabs -> column blocks) -> column FFT,
           x multiplier, inverse column FFT (local) -> all-to-all back -> inverse rows FFT
           -> u0 = max(Wiener, floor), fpos = max(f, floor)                (deconv.py:660-672)
  then ``iterations`` x:  halo exchange of u (periodic neighbours, matching the FOURIER_2D
           convolver's wrap, deconv.py:359-376) -> one RRRL iteration on the slab
           (direct taps, TV with Neumann boundary at the GLOBAL first/last row only)

Communication is only the halo rows (NCCL send/recv to rank +-1 mod world) and the two
spectrum transposes of the Wiener step (all-to-all). ``DistComm`` uses torch.distributed
(NCCL on GPUs, gloo on CPU); ``LocalComm`` runs the same SPMD code with one thread per
"rank" inside one process (host-side barriers and copies, no kernel waits on another), which
is how the decomposition is exercised on a single GPU.

Compute is delegated to a backend: ``CudaSlabBackend`` calls the C ABI (md_slab_*); tests may
plug in a NumPy backend to check the decomposition logic on CPU.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _lib as L

__all__ = ["SlabGeometry", "DistComm", "HostStagedComm", "LocalComm", "CudaSlabBackend", "SlabWorker", "run_slabs"]


class SlabGeometry:
    def __init__(self, H: int, W: int, rank: int, world: int, top: int, bottom: int):
        if H % world or W % world:
            raise ValueError("image height and width must divide by the number of ranks")
        self.H, self.W, self.rank, self.world = H, W, rank, world
        self.S = H // world
        self.Wb = W // world
        self.top, self.bottom = top, bottom
        if top > self.S or bottom > self.S:
            raise ValueError("slabs thinner than the PSF halo")
        self.row0 = rank * self.S

    @property
    def ext_rows(self) -> int:
        return self.top + self.S + self.bottom


# ---------------------------------------------------------------------------------- comms

class DistComm:
    """torch.distributed collectives (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

    def exchange(self, rank, send_up, send_down, recv_up, recv_down):
        """send_up -> rank-1 (its bottom halo); send_down -> rank+1 (its top halo); periodic."""
        dist = self.dist
        prev, nxt = (self.rank - 1) % self.world, (self.rank + 1) % self.world
        self.exchange_async(rank, send_up, send_down, recv_up, recv_down)()

    def exchange_async(self, rank, send_up, send_down, recv_up, recv_down):
        """Post the halo exchange; returns a wait() callable. On NCCL the transfers run on the
        communicator's stream while the caller's stream computes; wait() orders the caller's
        stream after them."""
        dist = self.dist
        prev, nxt = (self.rank - 1) % self.world, (self.rank + 1) % self.world
        if self.world == 1:
            recv_up.copy_(send_down)
            recv_down.copy_(send_up)
            return lambda: None
        ops = [dist.P2POp(dist.isend, send_up.contiguous(), prev, self.group),
               dist.P2POp(dist.irecv, recv_down, nxt, self.group),
               dist.P2POp(dist.isend, send_down.contiguous(), nxt, self.group),
               dist.P2POp(dist.irecv, recv_up, prev, self.group)]
        reqs = dist.batch_isend_irecv(ops)

        def wait():
            for req in reqs:
                req.wait()
        return wait

    def all_to_all(self, rank, recv, send):
        """send[q] goes to rank q, recv[q] comes from rank q (equal splits along dim 0)."""
        if self.world == 1:
            recv.copy_(send)
            return
        self.dist.all_to_all_single(recv, send, group=self.group)

    def barrier(self, rank):
        if self.world > 1:
            self.dist.barrier(self.group)


class HostStagedComm:
    """A DistComm over a backend that moves only host tensors (gloo): device buffers are
    staged through host copies around each exchange. Lets several processes share ONE GPU
    with a real process group -- the multi-process slab test (tests/test_gpu_slab_dist.py);
    on 8 GPUs NCCL moves device memory directly (DistComm)."""

    def __init__(self, comm: DistComm):
        self.c = comm
        self.rank, self.world = comm.rank, comm.world

    def exchange(self, rank, send_up, send_down, recv_up, recv_down):
        h = [t.detach().to("cpu").contiguous() for t in (send_up, send_down)]
        r_up, r_down = recv_up.new_empty(recv_up.shape, device="cpu"), recv_down.new_empty(recv_down.shape, device="cpu")
        self.c.exchange(rank, h[0], h[1], r_up, r_down)
        recv_up.copy_(r_up)
        recv_down.copy_(r_down)

    def exchange_async(self, rank, send_up, send_down, recv_up, recv_down):
        self.exchange(rank, send_up, send_down, recv_up, recv_down)      # host-side: done on return
        return lambda: None

    def all_to_all(self, rank, recv, send):
        r = recv.new_empty(recv.shape, device="cpu")
        self.c.all_to_all(rank, r, send.detach().to("cpu").contiguous())
        recv.copy_(r)

    def barrier(self, rank):
        self.c.barrier(rank)


class LocalComm:
    """All ranks as threads of one process; collectives = host barriers + tensor copies."""

    def __init__(self, world: int):
        self.world = world
        self._bar = threading.Barrier(world)
        self._box: dict = {}

    def exchange(self, rank, send_up, send_down, recv_up, recv_down):
        self._box[rank] = (send_up, send_down)
        self._bar.wait()
        prev, nxt = (rank - 1) % self.world, (rank + 1) % self.world
        recv_up.copy_(self._box[prev][1])       # prev's bottom rows -> my top halo
        recv_down.copy_(self._box[nxt][0])      # next's top rows -> my bottom halo
        self._bar.wait()

    def exchange_async(self, rank, send_up, send_down, recv_up, recv_down):
        self.exchange(rank, send_up, send_down, recv_up, recv_down)
        return lambda: None

    def all_to_all(self, rank, recv, send):
        self._box[rank] = send
        self._bar.wait()
        for q in range(self.world):
            recv[q].copy_(self._box[q][rank])
        self._bar.wait()

    def barrier(self, rank):
        self._bar.wait()


# ---------------------------------------------------------------------------------- backend

class CudaSlabBackend:
    """Per-rank compute through the C ABI (md_slab_*)."""

    def __init__(self, plan):
        self.plan = plan
        self.lib = plan.lib
        top, bot = ctypes.c_int32(), ctypes.c_int32()
        L.check(self.lib.md_slab_halo(plan._h, ctypes.byref(top), ctypes.byref(bot)))
        self.halo = (top.value, bot.value)
        self._mult = None

    def halo_rows(self):
        return self.halo

    def prepare(self, geo: SlabGeometry):
        ptr = ctypes.c_void_p()
        L.check(self.lib.md_slab_prepare(self.plan._h, geo.rank * geo.Wb, geo.Wb, ctypes.byref(ptr)))
        self._mult = ptr

    def rows_fft(self, z, real_in, rows, inv, scale=1.0, stream=None):
        L.check(self.lib.md_slab_rows_fft(self.plan._h, z.data_ptr(), None if real_in is None else real_in.data_ptr(),
                                          rows, inv, scale, _sp(stream)))

    def cols_filter(self, zc, cols, stream=None):
        L.check(self.lib.md_slab_cols_filter(self.plan._h, zc.data_ptr(), cols, self._mult, _sp(stream)))

    def epilogue(self, z, f, u0, fpos, rows, stream=None):
        L.check(self.lib.md_slab_wiener_epilogue(self.plan._h, z.data_ptr(), f.data_ptr(), u0.data_ptr(),
                                                 fpos.data_ptr(), rows, _sp(stream)))

    def bands(self):
        """(a_in, b_in): stage-A rows [a_in, S - a_in) and stage-B rows [b_in, S - b_in) need no
        halo rows (md_slab_bands)."""
        a, b, t, u = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        L.check(self.lib.md_slab_bands(self.plan._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(t),
                                       ctypes.byref(u)))
        self.adj_halo = (t.value, u.value)
        return a.value, b.value

    def stage(self, u_ext, fpos_ext, p_ext, w_ext, out_ext, geo: SlabGeometry, a_rows, b_rows, stream=None):
        """Part of one iteration: stage A over rows a_rows = (begin, end) of [-adj.ht, S + adj.hb),
        stage B over own rows b_rows (md_slab_stage)."""
        off = geo.top * geo.W * u_ext.element_size()
        ptr = lambda t: t.data_ptr() + off
        L.check(self.lib.md_slab_stage(self.plan._h, ptr(u_ext), ptr(fpos_ext), ptr(p_ext), ptr(w_ext),
                                       ptr(out_ext), geo.S, geo.row0, a_rows[0], a_rows[1], b_rows[0], b_rows[1],
                                       _sp(stream)))

    def iterate(self, u_ext, fpos_ext, p_ext, w_ext, out_ext, geo: SlabGeometry, stream=None):
        """One iteration on haloed [top + S + bottom, W] buffers (pointers at own row 0)."""
        off = geo.top * geo.W * u_ext.element_size()
        ptr = lambda t: t.data_ptr() + off
        L.check(self.lib.md_slab_iterate(self.plan._h, ptr(u_ext), ptr(fpos_ext), ptr(p_ext), ptr(w_ext),
                                         ptr(out_ext), geo.S, geo.row0, _sp(stream)))


def _sp(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream or None


# ---------------------------------------------------------------------------------- worker

class SlabWorker:
    """Buffers and SPMD program of one rank. ``f_own`` is this rank's [S, W] slab."""

    def __init__(self, backend, geo: SlabGeometry, iterations: int, device, dtype):
        import torch
        if not geo.top or not geo.bottom:
            raise ValueError("halo rows missing")
        self.b, self.g, self.K = backend, geo, iterations
        self.device, self.dtype = device, dtype
        g = geo
        ext = (g.ext_rows, g.W)
        self.u = [torch.zeros(ext, dtype=dtype, device=device) for _ in range(2)]
        self.fpos = torch.zeros(ext, dtype=dtype, device=device)
        self.p = torch.zeros(ext, dtype=dtype, device=device)
        self.w = torch.zeros(ext, dtype=dtype, device=device)
        self.z = torch.zeros((g.S, g.W, 2), dtype=dtype, device=device)          # complex as (re, im)
        self.send = torch.zeros((g.world, g.S, g.Wb, 2), dtype=dtype, device=device)
        self.recv = torch.zeros_like(self.send)
        backend.prepare(geo)

    def own(self, t):
        return t[self.g.top:self.g.top + self.g.S]

    def _exchange(self, comm, t):
        g = self.g
        # my first `bottom` rows feed rank-1's bottom halo; my last `top` rows feed rank+1's top halo
        comm.exchange(g.rank, self.own(t)[:g.bottom], self.own(t)[g.S - g.top:],
                      t[:g.top], t[g.top + g.S:])

    def run(self, comm, f_own):
        g, b = self.g, self.b
        # ---- Wiener: rows (local) -> transpose -> columns x M -> transpose back -> rows
        # the column block arrives as [world][S][Wb] = [H][Wb]: filtered in place in the receive
        # buffer and sent back from it (no staging copies around the column pass)
        b.rows_fft(self.z, f_own, g.S, 0)
        self.send.copy_(self.z.view(g.S, g.world, g.Wb, 2).permute(1, 0, 2, 3))
        comm.all_to_all(g.rank, self.recv, self.send)
        b.cols_filter(self.recv.view(g.H, g.Wb, 2), g.Wb)
        comm.all_to_all(g.rank, self.send, self.recv)
        self.z.view(g.S, g.world, g.Wb, 2).copy_(self.send.permute(1, 0, 2, 3))
        b.rows_fft(self.z, None, g.S, 1)
        cur = 0
        b.epilogue(self.z, f_own, self.own(self.u[cur]), self.own(self.fpos), g.S)
        self._exchange(comm, self.fpos)
        # ---- iterations. With a backend that runs stages by row band (CudaSlabBackend), the
        # rows that need no halo are computed while the halo exchange is in flight: stage A on
        # [a_in, S - a_in) and stage B on [b_in, S - b_in) first, then the boundary bands after
        # the exchange (on NCCL the transfer overlaps the interior kernels). Otherwise exchange,
        # then the whole iteration.
        bands = b.bands() if hasattr(b, "bands") else None
        ha_t, ha_b = getattr(b, "adj_halo", (None, None))
        overlap = bands is not None and 2 * bands[1] <= g.S and ha_t is not None
        for k in range(self.K):
            nxt = 1 - cur
            if overlap:
                a_in, b_in = bands
                t = self.u[cur]
                wait = comm.exchange_async(g.rank, self.own(t)[:g.bottom], self.own(t)[g.S - g.top:],
                                           t[:g.top], t[g.top + g.S:])
                b.stage(self.u[cur], self.fpos, self.p, self.w, self.u[nxt], g, (a_in, g.S - a_in),
                        (b_in, g.S - b_in))
                wait()
                for ar, br in (((-ha_t, a_in), (0, b_in)), ((g.S - a_in, g.S + ha_b), (g.S - b_in, g.S))):
                    b.stage(self.u[cur], self.fpos, self.p, self.w, self.u[nxt], g, ar, (0, 0))
                    b.stage(self.u[cur], self.fpos, self.p, self.w, self.u[nxt], g, (0, 0), br)
            else:
                self._exchange(comm, self.u[cur])
                b.iterate(self.u[cur], self.fpos, self.p, self.w, self.u[nxt], g)
            cur = nxt
        return self.own(self.u[cur])


def run_slabs(plan, f, world: int, backend_factory=CudaSlabBackend):
    """Deblur one [H, W] device image as ``world`` row slabs inside this process (LocalComm,
    one thread per slab). Returns the assembled [H, W] result."""
    import torch
    H, W = f.shape
    comm = LocalComm(world)
    out = torch.empty_like(f)
    errors = []
    backend = backend_factory(plan)
    top, bottom = backend.halo_rows()
    workers = [SlabWorker(backend_factory(plan) if r else backend, SlabGeometry(H, W, r, world, top, bottom),
                          plan.params.iterations, f.device, f.dtype) for r in range(world)]
    S = H // world

    def body(r):
        try:
            torch.cuda.set_device(f.device)
            res = workers[r].run(comm, f[r * S:(r + 1) * S].contiguous())
            torch.cuda.synchronize()
            out[r * S:(r + 1) * S].copy_(res)
            torch.cuda.synchronize()
        except BaseException as exc:            # surface worker failures, release the others
            errors.append(exc)
            comm._bar.abort()

    threads = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return out
