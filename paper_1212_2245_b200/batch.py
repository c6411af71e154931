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

    def run(self, frames, psf_index, out=None, stream=None):
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
        for b, s, e in self.groups(idx[order]):
            self.pipes[b].plan.run(src[s:e], out=dst[s:e], stream=stream)
        if sorted_already:
            return dst
        res = torch.empty_like(dst) if out is None else out
        res[torch.from_numpy(order).to(frames.device)] = dst
        return res

    def launch_count(self, psf_index) -> int:
        idx = np.sort(np.asarray(psf_index))
        return sum(self.pipes[b].plan.launch_count(e - s) for b, s, e in self.groups(idx))
