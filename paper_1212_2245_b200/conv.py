"""Spatial / box / Fourier convolution of one image on the B200 (conv.py, fft.py of the
reference): thin wrappers over the convolver realisations of the CUDA library.

``spatial_convolve`` -- clamped direct summation (conv.py:75-116); ``box_convolve`` -- clamped
O(1)-per-pixel sliding window (conv.py:119-135, 141-173); ``fourier_convolve`` -- periodic
convolution (fft.py:283-307), realised by direct wrap-around taps or 2D FFTs.
"""

from __future__ import annotations

import numpy as np

from .core import BlurAxis, Image, Psf, PsfKind, materialize_box_kernel
from .deconv import _dev, _image, make_convolver

__all__ = ["spatial_convolve", "box_convolve", "fourier_convolve", "convolve_array", "box_filter_array"]


def _check_support(psf: Psf, shape) -> None:
    sy, sx = psf.support
    if sy > shape[0] or sx > shape[1]:
        raise ValueError(f"PSF support {psf.support} exceeds image dimensions {shape}")


def spatial_convolve(image: Image, psf: Psf) -> Image:
    """Direct summation with edge-replicating boundaries (conv.py:75-82)."""
    _check_support(psf, image.shape)
    c = make_convolver(psf, image.shape, "spatial")
    return _image(c._plan.convolve(_dev(image), 0))


def box_convolve(image: Image, psf: Psf) -> Image:
    """Uniform-box convolution via sliding-window updates (conv.py:119-135)."""
    if psf.kind is not PsfKind.UNIFORM_BOX_1D:
        raise ValueError("box_convolve requires a uniform-box PSF")
    _check_support(psf, image.shape)
    c = make_convolver(psf, image.shape, "box")
    return _image(c._plan.convolve(_dev(image), 0))


def fourier_convolve(image: Image, psf: Psf, plans=None) -> Image:
    """Circular convolution (fft.py:283-307); transformed axes must be powers of two."""
    h, w = image.shape
    if psf.kind is PsfKind.GENERAL_2D:
        if not (_pow2(h) and _pow2(w)):
            raise ValueError("2D Fourier convolution needs power-of-two dimensions")
    elif not _pow2(h if psf.axis is BlurAxis.VERTICAL else w):
        raise ValueError("the blur axis must have power-of-two extent")
    c = make_convolver(psf, image.shape, "fourier2d" if psf.kind is PsfKind.GENERAL_2D else "fourier")
    return _image(c._plan.convolve(_dev(image), 0))


def _pow2(n: int) -> bool:
    return n >= 1 and n & (n - 1) == 0


def convolve_array(a: np.ndarray, psf: Psf) -> np.ndarray:
    """Array-level direct-summation convolution (conv.py:85-116; see spatial_convolve)."""
    return spatial_convolve(Image(np.asarray(a, dtype=np.float64)), psf).values


def box_filter_array(a: np.ndarray, length: float, center: int, axis: int = 0) -> np.ndarray:
    """Array-level box filter of ``length`` with the given tap ``center`` along ``axis``
    (conv.py:131-138): the clamped sliding-window convolver."""
    w = materialize_box_kernel(length)
    psf = Psf(PsfKind.UNIFORM_BOX_1D, w, int(center), axis=BlurAxis.VERTICAL if axis == 0 else BlurAxis.HORIZONTAL,
              length=float(length))
    return box_convolve(Image(np.asarray(a, dtype=np.float64)), psf).values
