"""``rrrl_deblur_parallel`` / ``ColumnSharpeningEngine`` (parallel.py:43-142 of the reference):
a COMPATIBILITY SHIM, not a parallel engine of its own.

The reference splits each RRRL iteration's columns over persistent host threads and guarantees
the serial result for any worker count (parallel.py:10-13). That thread engine is out of scope
here (the GPU replaces it). These entries keep the reference's signatures,
argument checks and orientation rules and run the ordinary device path: mode strings / None go
through ``rrrl_deblur`` (the fused kernels), a convolver object through the device step path
(deconv._iterate_steps, the object's own blur / adjoint_pair called with host arrays).
``workers`` / ``worker_count`` are validated and otherwise unused -- the result cannot depend on
them.
"""

from __future__ import annotations

import numpy as np

from .core import BlurAxis, DeconvParams, Image, Psf, PsfKind
from .deconv import (_clamp_dev, _convolver, _dev, _host, _iterate_steps, default_divergence_lut, rrrl_deblur)

__all__ = ["rrrl_deblur_parallel", "ColumnSharpeningEngine"]


class ColumnSharpeningEngine:
    """Same constructor and ``run`` as the reference's engine (parallel.py:43-114):
    ``run(u0, fpos, convolver, iterations, iteration_ms)`` applies ``iterations`` RRRL updates
    (_iterate_rrrl semantics: floored weights) to ``u0`` against ``fpos`` with ``convolver``
    (a ``make_convolver`` device convolver or any object with the protocol) on the device."""

    def __init__(self, params: DeconvParams, lut, workers: int):
        if workers < 1:
            raise ValueError("worker count must be at least 1")
        self.params = params
        self.lut = lut if lut is not None else default_divergence_lut()
        self.workers = int(workers)

    def run(self, u0: np.ndarray, fpos: np.ndarray, convolver, iterations: int,
            iteration_ms: list[float] | None = None) -> np.ndarray:
        if iterations <= 0:
            return u0
        conv = _convolver(None, np.shape(u0), convolver)
        return _host(self._loop(_dev(u0), _dev(fpos), conv, iterations, iteration_ms))

    def _loop(self, u, fp, conv, iterations, iteration_ms=None):
        import torch
        for _ in range(iterations):
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            u = _iterate_steps(u, fp, conv, self.params, self.lut)
            t1.record()
            if iteration_ms is not None:
                t1.synchronize()
                iteration_ms.append(t0.elapsed_time(t1))
        return u


def rrrl_deblur_parallel(f: Image, h: Psf, params: DeconvParams, worker_count: int = 1, *, convolver=None,
                         dtype: str = "float64") -> Image:
    """RRRL from the clamped input with a 1D PSF (parallel.py:117-142): uniform boxes use the
    sliding-window convolver, general 1D kernels the per-column (periodic) one unless
    ``convolver`` says otherwise. As in the reference, a convolver OBJECT sees the frame in
    vertical orientation (horizontal kernels are transposed around the call)."""
    if not h.is_1d:
        raise ValueError("parallel RRRL requires a 1D PSF")
    if worker_count < 1:
        raise ValueError("worker count must be at least 1")
    if convolver is None or isinstance(convolver, str):
        mode = convolver or ("box" if h.kind is PsfKind.UNIFORM_BOX_1D else "fourier")
        return rrrl_deblur(f, h, params, convolver=mode, dtype=dtype)
    transpose = h.axis is BlurAxis.HORIZONTAL
    a = np.ascontiguousarray(f.values.T) if transpose else f.values
    fp = _clamp_dev(_dev(a, dtype), params.floor)                       # np.maximum(a, floor)
    engine = ColumnSharpeningEngine(params, None, worker_count)
    u = _host(engine._loop(fp.clone(), fp, _convolver(None, a.shape, convolver, dtype), params.iterations))
    return Image._wrap(np.ascontiguousarray(u.T) if transpose else u)
