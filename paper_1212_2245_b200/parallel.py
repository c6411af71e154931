"""``rrrl_deblur_parallel`` (parallel.py:117-142 of the reference) on the B200.

The reference splits the RRRL sharpening columns across host threads and guarantees the same
result for any worker count. Here the GPU is the parallel engine: the call runs the serial
device path with the same convolver, so the result is independent of ``worker_count`` by
construction (the argument is validated, as in the reference, and otherwise unused).
"""

from __future__ import annotations

from .core import DeconvParams, Image, Psf, PsfKind
from .deconv import rrrl_deblur

__all__ = ["rrrl_deblur_parallel"]


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
