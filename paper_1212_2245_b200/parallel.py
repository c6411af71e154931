"""``rrrl_deblur_parallel`` (parallel.py:117-142 of the reference) on the B200.

The reference splits the RRRL sharpening columns across host threads and guarantees the same
result for any worker count. Here the GPU is the parallel engine: the call runs the serial
device path with the same convolver, so the result is independent of ``worker_count`` by
construction (the argument is validated, as in the reference, and otherwise unused).
"""

from __future__ import annotations

import time

import numpy as np

from .core import DeconvParams, Image, Psf, PsfKind
from .deconv import GpuConvolver, prepare_state, rrrl_deblur, rrrl_step

__all__ = ["rrrl_deblur_parallel", "ColumnSharpeningEngine"]


class ColumnSharpeningEngine:
    """The reference's threaded RRRL iteration engine (parallel.py:43-114) with the same
    interface, iterating on the device: ``run(u0, fpos, convolver, iterations, iteration_ms)``
    applies ``iterations`` RRRL updates to ``u0`` against the floored observation ``fpos`` with a
    device convolver (``GpuConvolver`` from ``make_convolver``); ``workers`` is validated as in
    the reference and otherwise unused (the GPU is the parallel engine)."""

    def __init__(self, params: DeconvParams, lut, workers: int):
        if workers < 1:
            raise ValueError("worker count must be at least 1")
        self.params = params
        self.lut = lut
        self.workers = int(workers)

    def run(self, u0: np.ndarray, fpos: np.ndarray, convolver, iterations: int,
            iteration_ms: list[float] | None = None) -> np.ndarray:
        if iterations <= 0:
            return u0
        if not isinstance(convolver, GpuConvolver):
            raise TypeError("ColumnSharpeningEngine.run needs a device convolver (make_convolver)")
        import torch
        u, f = Image(u0), Image(fpos)
        for _ in range(iterations):
            t0 = time.perf_counter()
            st = prepare_state(u, f, convolver.psf, self.params, convolver=convolver, lut=self.lut)
            u = rrrl_step(st, f, convolver.psf, self.params, convolver=convolver)
            if iteration_ms is not None:
                torch.cuda.synchronize()
                iteration_ms.append(1e3 * (time.perf_counter() - t0))
        return np.array(u.values)


def rrrl_deblur_parallel(f: Image, h: Psf, params: DeconvParams, worker_count: int = 1, *, convolver=None,
                         dtype: str = "float64") -> Image:
    """RRRL from the clamped input with a 1D PSF; uniform boxes use the sliding-window
    convolver, general 1D kernels the per-column (periodic) one unless ``convolver`` says
    otherwise (parallel.py:117-136)."""
    if not h.is_1d:
        raise ValueError("parallel RRRL requires a 1D PSF")
    if worker_count < 1:
        raise ValueError("worker count must be at least 1")
    if convolver is None:
        convolver = "box" if h.kind is PsfKind.UNIFORM_BOX_1D else "fourier"
    return rrrl_deblur(f, h, params, convolver=convolver, dtype=dtype)
