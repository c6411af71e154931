"""Batches of frames with a bank of PSFs (BASELINE.json configs[3], the "c4" workload).

Each frame carries the index of its PSF in a bank; frames sharing a PSF run as one batch
through that PSF's device plan (one ``DeblurPipeline`` per bank entry, scenario chosen as
the reference's ``default_scenario``, deconv.py:574-579). Frames are independent, so a
bank batch shards across GPUs by frame ranges with no collective.
"""

from __future__ import annotations

import numpy as np

from .core import DeconvParams, Psf
from .deconv import DeblurPipeline, Scenario, default_scenario

__all__ = ["PsfBankPipeline"]


class PsfBankPipeline:
    """Wiener + RRRL for frames blurred by different (known) PSFs of a bank.

    ``run(frames, psf_index)`` takes device frames ``[N, H, W]`` and per-frame bank indices;
    frames are grouped by PSF (a no-op when ``psf_index`` is already sorted), each group runs
    through its own plan, and results come back in the input order.
    """

    def __init__(self, shape, psfs: list[Psf], params: DeconvParams, dtype: str = "float32",
                 scenarios: list[Scenario] | None = None, chunk: int = 512):
        self.shape = tuple(shape)
        self.psfs = list(psfs)
        self.scenarios = scenarios or [default_scenario(p) for p in self.psfs]
        self.pipes = [DeblurPipeline(self.shape, p, params, s, dtype=dtype)
                      for p, s in zip(self.psfs, self.scenarios)]
        for p in self.pipes:
            p.plan.set_chunk(chunk)          # bound per-plan scratch: the bank shares one device

    def groups(self, psf_index: np.ndarray) -> list[tuple[int, int, int]]:
        """(bank entry, start, stop) runs of a sorted index vector."""
        idx = np.asarray(psf_index)
        if idx.size and np.any(np.diff(idx) < 0):
            raise ValueError("psf_index must be sorted (use run(), which sorts)")
        out, start = [], 0
        for i in range(1, idx.size + 1):
            if i == idx.size or idx[i] != idx[start]:
                out.append((int(idx[start]), start, i))
                start = i
        return out

    def run(self, frames, psf_index, out=None, stream=None, streams: int = 1):
        """``streams`` > 1 deals the PSF groups round-robin over that many internal CUDA streams
        (ordered after, and joined back into, the caller's stream), so one group's last
        partial wave of clusters overlaps the next group's launches."""
        import torch
        idx = np.asarray(psf_index, dtype=np.int64)
        if frames.shape[0] != idx.size:
            raise ValueError("one PSF index per frame")
        if idx.size and (idx.min() < 0 or idx.max() >= len(self.pipes)):
            raise ValueError("PSF index out of range")
        order = np.argsort(idx, kind="stable")
        sorted_already = bool(np.all(order == np.arange(idx.size)))
        src = frames if sorted_already else frames[torch.from_numpy(order).to(frames.device)]
        dst = (out if (out is not None and sorted_already) else torch.empty_like(src))
        groups = self.groups(idx[order])
        if streams > 1 and len(groups) > 1:
            base = stream if stream is not None else torch.cuda.current_stream()
            if len(getattr(self, "_run_streams", ())) != streams:
                self._run_streams = [torch.cuda.Stream() for _ in range(streams)]
            for st in self._run_streams:
                st.wait_stream(base)
            for k, (b, s, e) in enumerate(groups):
                self.pipes[b].plan.run(src[s:e], out=dst[s:e], stream=self._run_streams[k % streams])
            for st in self._run_streams:
                base.wait_stream(st)
        else:
            for b, s, e in groups:
                self.pipes[b].plan.run(src[s:e], out=dst[s:e], stream=stream)
        if sorted_already:
            return dst
        res = torch.empty_like(dst) if out is None else out
        res[torch.from_numpy(order).to(frames.device)] = dst
        return res

    def run_host(self, frames, psf_index, out=None, out_dtype=np.float32, max_piece: int = 512):
        """Host frames (uint8 / float32 / float64 ``[N, H, W]``) -> host results (float32 / float64,
        or uint8 with the reference's write_pgm quantisation), pipelined across
        PSF groups: the host->device copy of group g+1 and the device->host copy of group g-1
        overlap the deconvolution of group g (three CUDA streams, events between them). Pinned
        (page-locked) host arrays make the copies asynchronous."""
        import torch
        from .plan import convert_dev, torch_dtype
        a = np.asarray(frames)
        idx = np.asarray(psf_index, dtype=np.int64)
        if a.ndim != 3 or a.shape[1:] != self.shape or a.shape[0] != idx.size:
            raise ValueError(f"frames must be [N, {self.shape[0]}, {self.shape[1]}] with one PSF index each")
        if a.dtype not in (np.uint8, np.float32, np.float64):
            a = a.astype(np.float64)
        if idx.size and (idx.min() < 0 or idx.max() >= len(self.pipes)):
            raise ValueError("PSF index out of range")
        order = np.argsort(idx, kind="stable")
        sorted_already = bool(np.all(order == np.arange(idx.size)))
        if not sorted_already:
            a, idx = a[order], idx[order]
        a = np.ascontiguousarray(a)
        n = a.shape[0]
        res = np.empty(a.shape, dtype=out_dtype) if (out is None or not sorted_already) else out
        if res.dtype not in (np.float32, np.float64, np.uint8) or res.shape != a.shape or not res.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float32/float64/uint8 array of the frames' shape")
        pdt = torch_dtype(self.pipes[0].dtype)
        odt = torch.from_numpy(np.zeros(1, res.dtype)).dtype
        key = (n, a.dtype.str, res.dtype.str)
        if getattr(self, "_host_key", None) != key:         # device staging, reused across calls
            hin_t = torch.from_numpy(a[:1]).dtype
            dev = torch.device("cuda")
            self._dbuf = {"in": torch.empty(a.shape, dtype=hin_t, device=dev),
                          "f": torch.empty(a.shape, dtype=pdt, device=dev),
                          "u": torch.empty(a.shape, dtype=pdt, device=dev),
                          "o": torch.empty(a.shape, dtype=odt, device=dev) if odt != pdt else None}
            self._streams = [torch.cuda.Stream() for _ in range(3)]
            self._host_key = key
        d = self._dbuf
        h2d, cmp, d2h = self._streams
        hin, hout = torch.from_numpy(a), torch.from_numpy(res)
        din = d["in"]
        dfin = din if din.dtype == pdt else d["f"]
        dres = d["o"] if d["o"] is not None else d["u"]
        pieces = []
        for b, s, e in self.groups(idx):
            for p0 in range(s, e, max_piece):
                pieces.append((b, p0, min(e, p0 + max_piece)))
        cur = torch.cuda.current_stream()
        for st in (h2d, cmp, d2h):
            st.wait_stream(cur)
        for b, s, e in pieces:
            with torch.cuda.stream(h2d):
                din[s:e].copy_(hin[s:e], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(h2d)
            cmp.wait_event(ev)
            if dfin is not din:
                convert_dev(din[s:e], dfin[s:e], stream=cmp)
            self.pipes[b].plan.run(dfin[s:e], out=d["u"][s:e], stream=cmp)
            if dres is not d["u"]:
                convert_dev(d["u"][s:e], dres[s:e], stream=cmp)
            ev = torch.cuda.Event()
            ev.record(cmp)
            d2h.wait_event(ev)
            with torch.cuda.stream(d2h):
                hout[s:e].copy_(dres[s:e], non_blocking=True)
        d2h.synchronize()
        if sorted_already:
            return res
        dst = np.empty(res.shape, dtype=res.dtype) if out is None else out
        dst[order] = res
        return dst

    def launch_count(self, psf_index) -> int:
        idx = np.sort(np.asarray(psf_index))
        return sum(self.pipes[b].plan.launch_count(e - s) for b, s, e in self.groups(idx))
