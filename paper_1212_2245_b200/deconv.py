"""Wiener filtering, RL / RRRL and the Wiener + RRRL pipeline -- on the B200.

Same public names, signatures, defaults and exceptions as the reference module
``motiondeblur/deconv.py`` (drop-in), with every pixel operation executed by the CUDA
library through ``GpuPlan``. ``Image`` arguments are host float64 grids as in the
reference; the batched entry ``DeblurPipeline.run_batch`` takes and returns device
tensors ``[N, H, W]`` (or host arrays, staged through the C-ABI host entry).

Reference anchors are given per function. The update implemented by the kernels is

    u' = u * [ (W f / (u*h)) * h~ + alpha pos(D) ] / max(W * h~ - alpha neg(D), 1e-12)

with W = 0.5 / sqrt(f r1((u*h)/f) + eps_d^2) from the interpolated divergence table and
D the Neumann TV divergence (deconv.py:1-25).
"""

from __future__ import annotations

import enum
import functools
import math
from dataclasses import dataclass

import numpy as np

from .core import (DEFAULT_FLOOR, BlurAxis, ContractError, DeconvParams, Image, Psf, PsfKind)
from .plan import GpuPlan, device_min, diffusion_dev, guard_, robust_weight_dev, torch_dtype

__all__ = [
    "DIVISION_GUARD", "DivergenceLut", "default_divergence_lut", "robust_weight", "diffusion_term",
    "diffusion_energy", "wiener_2d", "wiener_1d", "rl_step", "rl_deblur", "SharpeningState",
    "prepare_state", "rrrl_step", "rrrl_deblur", "Scenario", "default_scenario", "make_convolver",
    "StageTimes", "DeblurPipeline", "wr3l",
]

DIVISION_GUARD = 1e-12      # deconv.py:74


# ------------------------------------------------------------------------------------------
# plan cache (plans hold device tables; one-shot entry points reuse them)

def _psf_key(psf: Psf):
    return (psf.kind, psf.weights.shape, psf.weights.tobytes(), psf.center, psf.axis, psf.length)


@functools.lru_cache(maxsize=64)
def _cached_plan(shape, psf_key, psf_ref, params, conv, init, dtype, rl, force_fft2d):
    return GpuPlan(shape, psf_ref[0], params, conv, init=init, dtype=dtype, rl=rl, force_fft2d=force_fft2d)


def _unchecked_params(**fields) -> DeconvParams:
    """A DeconvParams carrying `fields` without its validation (callers whose reference
    counterpart does not validate, e.g. rl_deblur's floor)."""
    p = object.__new__(DeconvParams)
    for k, v in {**DeconvParams().__dict__, **fields}.items():
        object.__setattr__(p, k, v)
    return p


def _plan(shape, psf: Psf, params: DeconvParams, conv: str, init="wiener", dtype="float64", rl=False,
          force_fft2d=False) -> GpuPlan:
    # psf_ref is a 1-tuple so the Psf (unhashable by value) rides along without keying the cache
    return _cached_plan(tuple(int(s) for s in shape), _psf_key(psf), _Ref(psf), params, conv, init, dtype,
                        rl, force_fft2d)


class _Ref(tuple):
    """Wrapper that hashes/compares equal for any payload (the key already pins it)."""

    def __new__(cls, obj):
        return super().__new__(cls, (obj,))

    def __hash__(self):
        return 0

    def __eq__(self, other):
        return isinstance(other, _Ref)


def _dev(a, dtype="float64"):
    """Host image / array -> contiguous CUDA tensor of the plan dtype."""
    import torch
    if isinstance(a, Image):
        a = a.values
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch_dtype(dtype)).contiguous()
    a = np.ascontiguousarray(a, dtype=np.float64)
    if not a.flags.writeable:
        a = a.copy()
    return torch.from_numpy(a).to(device="cuda", dtype=torch_dtype(dtype)).contiguous()


def _host(t) -> np.ndarray:
    return t.detach().to("cpu").double().numpy()


def _image(t) -> Image:
    return Image._wrap(np.ascontiguousarray(_host(t)))


# ------------------------------------------------------------------------------------------
# divergence table (deconv.py:81-139). The table is built and evaluated on the device: the
# reference parameters are compiled into the pipeline kernels (md_common.cuh); any other
# parameters get a device table of their own (md_lut_build) evaluated with runtime parameters
# (md_lut_r1_custom / md_robust_weight_custom), and the entries that take a `lut` then run the
# iteration step by step (the fused kernels know only the default table).

_DEFAULT_LUT = (1.0 / 32.0, 1.0 / 2048.0, 65.0, 0.5)


@dataclass(frozen=True, eq=False)
class DivergenceLut:
    delta: float
    step: float
    upper: float
    direct_below: float
    linear_slope: float
    linear_intercept: float

    @classmethod
    def build(cls, delta: float = 1.0 / 32.0, step: float = 1.0 / 2048.0, upper: float = 65.0,
              direct_below: float = 0.5) -> "DivergenceLut":
        if not 0.0 < delta < direct_below < upper:
            raise ValueError("need 0 < delta < direct_below < upper")
        slope = 1.0 - 1.0 / upper
        return cls(delta, step, upper, direct_below, slope, (upper - 1.0 - math.log(upper)) - slope * upper)

    @property
    def count(self) -> int:
        return int(round((self.upper - self.delta) / self.step)) + 1      # deconv.py:104

    @property
    def is_default(self) -> bool:
        return (self.delta, self.step, self.upper, self.direct_below) == _DEFAULT_LUT

    def _device_table(self):
        """The custom table on the current device (built once per object and device)."""
        import torch
        from . import _lib as L
        dev = torch.cuda.current_device()
        cache = self.__dict__.setdefault("_tables", {})
        if dev not in cache:
            t = torch.empty(self.count, dtype=torch.float64, device="cuda")
            L.check(L.lib().md_lut_build(t.data_ptr(), t.numel(), self.delta, self.step, None))
            cache[dev] = t
        return cache[dev]

    def _args(self):
        t = self._device_table()
        return (t.data_ptr(), t.numel(), self.delta, self.step, self.upper, self.direct_below, self.linear_slope,
                self.linear_intercept)

    @property
    def table(self) -> np.ndarray:
        """The nodes x_i - 1 - ln x_i, built on the device (copied to the host)."""
        import ctypes
        from . import _lib as L
        if self.is_default:
            out = np.empty(133057)
            L.check(L.lib().md_lut_table(out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), out.size))
        else:
            out = _host(self._device_table())
        out.setflags(write=False)
        return out

    def r1(self, x) -> np.ndarray:
        """r1 by table interpolation with the linear / exact extensions, on the device, in the
        reference's rounding order."""
        from . import _lib as L
        from .plan import _stream_ptr
        xd = _dev(np.asarray(x, dtype=np.float64))
        out = xd.new_empty(xd.shape)
        if self.is_default:
            L.check(L.lib().md_lut_r1(L.MD_F64, xd.data_ptr(), out.data_ptr(), xd.numel(), _stream_ptr(None)))
        else:
            L.check(L.lib().md_lut_r1_custom(*self._args(), xd.data_ptr(), out.data_ptr(), xd.numel(),
                                             _stream_ptr(None)))
        return _host(out)

    def weight_dev(self, f, b, eps_data: float, floor: float, assume_floored: bool = False):
        """_weight_arrays (deconv.py:142-162) with this table, device tensors in and out."""
        if self.is_default:
            return robust_weight_dev(f, b, eps_data, floor, assume_floored)
        from . import _lib as L
        from .plan import _stream_ptr, dtype_code
        out = b.new_empty(b.shape)
        L.check(L.lib().md_robust_weight_custom(dtype_code(f), *self._args(), f.data_ptr(), b.data_ptr(),
                                                out.data_ptr(), f.numel(), eps_data, floor,
                                                1 if assume_floored else 0, _stream_ptr(None)))
        return out


@functools.lru_cache(maxsize=1)
def default_divergence_lut() -> DivergenceLut:
    return DivergenceLut.build()


def _require_positive(img, what: str) -> None:
    """deconv.py:410-412 -- min over the device copy."""
    if device_min(img) <= 0.0:
        raise ContractError(f"{what} must be strictly positive")


# ------------------------------------------------------------------------------------------
# robust weight and diffusion (deconv.py:142-246)

def robust_weight(f: Image, b: Image, lut: DivergenceLut | None = None, eps_data: float = 1.0,
                  floor: float = DEFAULT_FLOOR) -> Image:
    """W = phi'(r_f(b)), phi(z) = sqrt(z + eps^2); f < floor uses max(b - f, 0) (deconv.py:165-180)."""
    if f.shape != b.shape:
        raise ValueError("observation and blurred iterate must match in shape")
    bd = _dev(b)
    if device_min(bd) <= 0.0:
        raise ContractError("blurred iterate must be strictly positive")
    lut = default_divergence_lut() if lut is None else lut
    return _image(lut.weight_dev(_dev(f), bd, eps_data, floor))


def diffusion_term(u: Image, eps_reg: float) -> Image:
    """TV divergence div(psi'(|grad u|^2) grad u), Neumann boundary (deconv.py:216-228)."""
    if not eps_reg > 0.0:
        raise ValueError("eps_reg must be positive")
    return _image(diffusion_dev(_dev(u), eps_reg))


def diffusion_energy(u: Image, eps_reg: float) -> float:
    """sum sqrt(|grad u|^2 + eps^2) (deconv.py:231-246). A scalar diagnostic, evaluated on the
    host -- it is not part of the deblurring path."""
    a = u.values
    gx2 = np.diff(a, axis=1) ** 2
    gy2 = np.diff(a, axis=0) ** 2
    q = np.zeros_like(a)
    q[:, :-1] += gx2
    q[:, 1:] += gx2
    q[:-1, :] += gy2
    q[1:, :] += gy2
    return float(np.sum(np.sqrt(0.5 * q + eps_reg * eps_reg)))


# ------------------------------------------------------------------------------------------
# Wiener (deconv.py:253-288)

def wiener_2d(f: Image, h: Psf, k: float, plans=None, dtype: str = "float64") -> Image:
    """2D-FFT Wiener filter, unclamped (deconv.py:257-272); ``plans`` is accepted and unused."""
    if not k > 0.0:
        raise ValueError("Wiener filter parameter K must be positive")
    p = _plan(f.shape, h, DeconvParams(wiener_k=k, iterations=0), "fourier2d", dtype=dtype)
    return _image(p.wiener(_dev(f, dtype)))


def wiener_1d(f: Image, h: Psf, k: float, plan=None, dtype: str = "float64") -> Image:
    """Per-line Wiener filter for 1D kernels, unclamped (deconv.py:275-288)."""
    if not k > 0.0:
        raise ValueError("Wiener filter parameter K must be positive")
    if not h.is_1d:
        raise ValueError("wiener_1d requires a 1D PSF")
    p = _plan(f.shape, h, DeconvParams(wiener_k=k, iterations=0), "fourier", dtype=dtype)
    return _image(p.wiener(_dev(f, dtype)))


# ------------------------------------------------------------------------------------------
# convolvers (deconv.py:295-403)

class GpuConvolver:
    """Convolver protocol ``blur / adjoint / adjoint_pair`` (deconv.py:295-376) on the device.

    Accepts numpy arrays (returns numpy) or CUDA tensors (returns tensors, no host copy).
    """

    def __init__(self, psf: Psf, shape, mode: str, dtype: str = "float64"):
        self.psf, self.shape, self.mode, self.dtype = psf, tuple(shape), mode, dtype
        self._plan = _plan(shape, psf, DeconvParams(iterations=0), mode, init="clamped", dtype=dtype)

    def _apply(self, a, which):
        import torch
        t = a if isinstance(a, torch.Tensor) else _dev(a, self.dtype)
        out = self._plan.convolve(t, which)
        return out if isinstance(a, torch.Tensor) else _host(out)

    def blur(self, a):
        return self._apply(a, 0)

    def adjoint(self, a):
        return self._apply(a, 1)

    def adjoint_pair(self, p, q):
        import torch
        tp = p if isinstance(p, torch.Tensor) else _dev(p, self.dtype)
        tq = q if isinstance(q, torch.Tensor) else _dev(q, self.dtype)
        op, oq = self._plan.adjoint_pair(tp, tq)
        if isinstance(p, torch.Tensor):
            return op, oq
        return _host(op), _host(oq)


def make_convolver(psf: Psf, shape: tuple[int, int], mode: str | None = None, dtype: str = "float64"):
    """deconv.py:379-403 -- "spatial" | "box" | "fourier" | "fourier2d" | None (box for box
    kernels, clamped direct summation otherwise)."""
    if mode is None:
        mode = "box" if psf.kind is PsfKind.UNIFORM_BOX_1D else "spatial"
    if mode not in ("spatial", "box", "fourier", "fourier2d"):
        raise ValueError(f"unknown convolver mode {mode!r}")
    if mode == "box" and psf.kind is not PsfKind.UNIFORM_BOX_1D:
        raise ValueError("box convolver requires a uniform-box PSF")
    if mode == "fourier" and psf.kind is PsfKind.GENERAL_2D:
        mode = "fourier2d"
    return GpuConvolver(psf, shape, mode, dtype)


def _convolver(h: Psf, shape, convolver, dtype="float64"):
    """A mode string / None -> the device convolver; a GpuConvolver as is; any other object with
    the reference's convolver protocol (blur / adjoint / adjoint_pair on float64 arrays,
    deconv.py:295-376; accepted wherever the reference accepts one, deconv.py:456-457, 549-550)
    -> wrapped so it is called with host arrays while every other step stays on the device."""
    if convolver is None or isinstance(convolver, str):
        return make_convolver(h, shape, convolver, dtype)
    if isinstance(convolver, GpuConvolver):
        return convolver
    for name in ("blur", "adjoint", "adjoint_pair"):
        if not callable(getattr(convolver, name, None)):
            raise TypeError(f"convolver object lacks {name}() (the protocol of deconv.py:295-376)")
    return _ForeignConvolver(convolver, dtype)


class _ForeignConvolver:
    """A caller's convolver object behind device-tensor blur / adjoint / adjoint_pair: tensors go
    to the host as float64 arrays, through the object, and back. Only the object's own work runs
    where the object runs it; ratio, weights, diffusion and the update are device kernels."""

    def __init__(self, obj, dtype: str):
        self.obj, self.dtype = obj, dtype

    def blur(self, t):
        return _dev(np.asarray(self.obj.blur(_host(t)), dtype=np.float64), self.dtype)

    def adjoint(self, t):
        return _dev(np.asarray(self.obj.adjoint(_host(t)), dtype=np.float64), self.dtype)

    def adjoint_pair(self, p, q):
        a, b = self.obj.adjoint_pair(_host(p), _host(q))
        return _dev(np.asarray(a, dtype=np.float64), self.dtype), _dev(np.asarray(b, dtype=np.float64), self.dtype)


def _dev_ops(conv):
    """Device-tensor blur / adjoint / adjoint_pair of a GpuConvolver or a wrapped object."""
    if isinstance(conv, GpuConvolver):
        return (lambda t: conv._plan.convolve(t, 0), lambda t: conv._plan.convolve(t, 1),
                lambda p, q: conv._plan.adjoint_pair(p, q))
    return conv.blur, conv.adjoint, conv.adjoint_pair


# ------------------------------------------------------------------------------------------
# device step toolkit (deconv.py:415-446, 512-521) for the step-by-step paths: a caller's
# convolver object, or a DivergenceLut with non-default parameters

def _clamp_dev(t, floor: float):
    from . import _lib as L
    from .plan import _stream_ptr, dtype_code
    out = t.new_empty(t.shape)
    L.check(L.lib().md_clamp(dtype_code(t), t.data_ptr(), out.data_ptr(), t.numel(), float(floor), _stream_ptr(None)))
    return out


def _ratio_dev(f, b, w=None):
    from . import _lib as L
    from .plan import _stream_ptr, dtype_code
    out = b.new_empty(b.shape)
    L.check(L.lib().md_ratio(dtype_code(b), f.data_ptr(), b.data_ptr(), None if w is None else w.data_ptr(),
                             out.data_ptr(), b.numel(), _stream_ptr(None)))
    return out


def _combine_dev(u, num, den, d, alpha: float):
    """_combine's assembly (deconv.py:421-446): u (num + a D+) / max(den - a D-, 1e-12)."""
    from . import _lib as L
    from .plan import _stream_ptr, dtype_code
    out = u.new_empty(u.shape)
    L.check(L.lib().md_combine(dtype_code(u), u.data_ptr(), num.data_ptr(), None if den is None else den.data_ptr(),
                               None if d is None else d.data_ptr(), out.data_ptr(), u.numel(), float(alpha),
                               _stream_ptr(None)))
    return out


def _combine_steps(u, f, b, w, d, alpha, conv):
    """_combine (deconv.py:421-446) with the convolver's adjoint(s)."""
    _, adjoint, adjoint_pair = _dev_ops(conv)
    if w is None:
        return _combine_dev(u, adjoint(_ratio_dev(f, b)), None, d, alpha)
    num, den = adjoint_pair(_ratio_dev(f, b, w), w)
    return _combine_dev(u, num, den, d, alpha)


def _iterate_steps(u, fpos, conv, params: DeconvParams, lut: "DivergenceLut", robust: bool = True):
    """_iterate_rrrl (deconv.py:512-521), one device step at a time."""
    blur = _dev_ops(conv)[0]
    b = guard_(blur(u))
    w = lut.weight_dev(fpos, b, params.eps_data, params.floor, assume_floored=True) if robust else None
    d = diffusion_dev(u, params.eps_reg) if params.alpha > 0.0 else None
    return _combine_steps(u, fpos, b, w, d, params.alpha, conv)


def _stepwise(conv, lut) -> bool:
    return not isinstance(conv, GpuConvolver) or (lut is not None and not lut.is_default)


# ------------------------------------------------------------------------------------------
# RL / RRRL steps (deconv.py:449-559)

@dataclass(frozen=True, eq=False)
class SharpeningState:
    """Fields feeding one RRRL update (deconv.py:463-474)."""

    iterate: Image
    blurred: Image
    weight: Image | None
    diffusion: Image | None


def rl_step(u: Image, f: Image, h: Psf, convolver=None) -> Image:
    """u' = u * ((f / max(u*h, 1e-12)) * h~) (deconv.py:449-460)."""
    ud, fd = _dev(u), _dev(f)
    _require_positive(ud, "RL iterate")
    _require_positive(fd, "RL observation")
    conv = _convolver(h, u.shape, convolver)
    if not isinstance(conv, GpuConvolver):
        return _image(_combine_steps(ud, fd, guard_(conv.blur(ud)), None, None, 0.0, conv))
    b = guard_(conv._plan.convolve(ud, 0))
    return _image(conv._plan.rrrl_step(ud, fd, b))


def prepare_state(u: Image, f: Image, h: Psf, params: DeconvParams, convolver=None,
                  lut: DivergenceLut | None = None, robust: bool = True) -> SharpeningState:
    """Blurred iterate, robust weight and diffusion field (deconv.py:477-496)."""
    ud, fd = _dev(u), _dev(f)
    _require_positive(ud, "RRRL iterate")
    _require_positive(fd, "RRRL observation")
    conv = _convolver(h, u.shape, convolver)
    lut = default_divergence_lut() if lut is None else lut
    b = guard_(_dev_ops(conv)[0](ud))
    w = lut.weight_dev(fd, b, params.eps_data, params.floor) if robust else None
    d = diffusion_dev(ud, params.eps_reg) if params.alpha > 0.0 else None
    return SharpeningState(u, _image(b), None if w is None else _image(w), None if d is None else _image(d))


def rrrl_step(state: SharpeningState, f: Image, h: Psf, params: DeconvParams, convolver=None) -> Image:
    """One robust regularised RL update from a prepared state (deconv.py:499-509)."""
    ud = _dev(state.iterate)
    _require_positive(ud, "RRRL iterate")
    conv = _convolver(h, state.iterate.shape, convolver)
    w = None if state.weight is None else _dev(state.weight)
    d = None if state.diffusion is None else _dev(state.diffusion)
    if not isinstance(conv, GpuConvolver):
        return _image(_combine_steps(ud, _dev(f), _dev(state.blurred), w, d, params.alpha, conv))
    out = conv._plan.rrrl_step(ud, _dev(f), _dev(state.blurred), w, d, alpha=params.alpha)
    return _image(out)


def rl_deblur(f: Image, h: Psf, iterations: int, convolver=None, floor: float = DEFAULT_FLOOR,
              dtype: str = "float64") -> Image:
    """Richardson-Lucy from the clamped input (deconv.py:524-534). As in the reference the
    iteration count is a ``range`` bound (non-integers raise TypeError, negative counts run
    none) and ``floor`` is only the clamp value: no DeconvParams validation applies."""
    count = len(range(iterations))
    conv = _convolver(h, f.shape, convolver, dtype)
    if not isinstance(conv, GpuConvolver):
        fpos = _clamp_dev(_dev(f, dtype), floor)
        u = fpos.clone()
        for _ in range(count):
            u = _combine_steps(u, fpos, guard_(conv.blur(u)), None, None, 0.0, conv)
        return _image(u)
    params = _unchecked_params(iterations=count, floor=float(floor))
    p = _plan(f.shape, h, params, conv.mode, init="clamped", dtype=dtype, rl=True)
    return _image(p.run(_dev(f, dtype)))


def rrrl_deblur(f: Image, h: Psf, params: DeconvParams, convolver=None,
                lut: DivergenceLut | None = None, dtype: str = "float64") -> Image:
    """RRRL from the clamped input (deconv.py:537-559); default convolver is box for box
    kernels and clamped direct summation otherwise. A caller's convolver object or a
    non-default divergence table runs the iterations step by step on the device."""
    conv = _convolver(h, f.shape, convolver, dtype)
    if _stepwise(conv, lut):
        lut = default_divergence_lut() if lut is None else lut
        fpos = _clamp_dev(_dev(f, dtype), params.floor)
        u = fpos.clone()
        for _ in range(params.iterations):
            u = _iterate_steps(u, fpos, conv, params, lut)
        return _image(u)
    p = _plan(f.shape, h, params, conv.mode, init="clamped", dtype=dtype)
    return _image(p.run(_dev(f, dtype)))


# ------------------------------------------------------------------------------------------
# the combined pipeline (deconv.py:566-703)

class Scenario(enum.Enum):
    """Algorithmic fast path for the blur at hand (deconv.py:566-571)."""

    BOX_1D = "box"
    FOURIER_1D = "fourier1d"
    FOURIER_2D = "fourier2d"


_SCENARIO_CONV = {Scenario.BOX_1D: "box", Scenario.FOURIER_1D: "fourier", Scenario.FOURIER_2D: "fourier2d"}


def default_scenario(psf: Psf) -> Scenario:
    """deconv.py:574-579."""
    if psf.kind is PsfKind.UNIFORM_BOX_1D:
        return Scenario.BOX_1D
    if psf.kind is PsfKind.GENERAL_1D:
        return Scenario.FOURIER_1D
    return Scenario.FOURIER_2D


@dataclass
class StageTimes:
    """Milliseconds per pipeline stage of one run (deconv.py:582-592), from CUDA events."""

    wiener_ms: float
    iteration_ms: list[float]
    total_ms: float

    @property
    def rrrl_total_ms(self) -> float:
        return sum(self.iteration_ms)


def _is_pow2(n: int) -> bool:
    return n >= 1 and n & (n - 1) == 0


class DeblurPipeline:
    """Prepared Wiener + RRRL pipeline for one frame shape (deconv.py:602-693).

    Construction builds the device plan (taps, twiddles, Wiener multiplier, divergence
    table); ``run``/``run_timed`` process one ``Image``; ``run_batch`` processes a stack of
    frames ``[N, H, W]`` resident on the device (or host, staged through md_run_host).
    ``workers`` is accepted for signature compatibility (the GPU replaces the thread engine).
    ``dtype`` selects the arithmetic ("float64" default, "float32" where parity allows).
    """

    def __init__(self, shape: tuple[int, int], psf: Psf, params: DeconvParams,
                 scenario: Scenario | None = None, workers: int = 1, lut: DivergenceLut | None = None,
                 dtype: str = "float64", fused: bool | None = None, force_fft2d: bool = False,
                 generic_lines: bool = False, big_fft: bool = False):
        if scenario is None:
            scenario = default_scenario(psf)
        if scenario in (Scenario.BOX_1D, Scenario.FOURIER_1D) and not psf.is_1d:
            raise ValueError(f"{scenario.name} requires a 1D PSF")
        if scenario is Scenario.BOX_1D and psf.kind is not PsfKind.UNIFORM_BOX_1D:
            raise ValueError("BOX_1D requires a uniform-box PSF")
        self.scenario = scenario
        self.params = params
        self.workers = int(workers)
        self.dtype = dtype
        self.shape = (int(shape[0]), int(shape[1]))
        sy, sx = psf.support
        if sy > self.shape[0] or sx > self.shape[1]:
            raise ValueError("PSF support exceeds the image dimensions")
        if scenario is Scenario.FOURIER_2D:
            if not (_is_pow2(self.shape[0]) and _is_pow2(self.shape[1])):
                raise ValueError("transform length must be a power of two")
        else:
            n = self.shape[0] if psf.axis is BlurAxis.VERTICAL else self.shape[1]
            if not _is_pow2(n):
                raise ValueError("the blur axis must have power-of-two extent")
        self.psf = psf
        self._plan = GpuPlan(self.shape, psf, params, _SCENARIO_CONV[scenario], init="wiener", dtype=dtype,
                             force_fft2d=force_fft2d, fused=fused, generic_lines=generic_lines,
                             big_fft=big_fft)
        self._wiener_plan = None
        # a non-default divergence table: the Wiener step through a 0-iteration plan, then the
        # iterations step by step with the scenario's device convolver (deconv.py:653-690)
        self.lut = lut
        self._steps = None
        if lut is not None and not lut.is_default:
            p0 = DeconvParams(params.wiener_k, params.alpha, 0, params.eps_data, params.eps_reg, params.floor)
            self._steps = (GpuPlan(self.shape, psf, p0, _SCENARIO_CONV[scenario], init="wiener", dtype=dtype,
                                   force_fft2d=force_fft2d, big_fft=big_fft),
                           make_convolver(psf, self.shape, _SCENARIO_CONV[scenario], dtype))

    def _run_steps(self, f):
        """Wiener -> clamp -> iterations with the custom table, device tensors [.., H, W]."""
        wplan, conv = self._steps
        u = wplan.run(f)
        fpos = _clamp_dev(f, self.params.floor)
        for _ in range(self.params.iterations):
            u = _iterate_steps(u, fpos, conv, self.params, self.lut)
        return u

    @property
    def plan(self) -> GpuPlan:
        return self._plan

    def _check_shape(self, shape):
        if tuple(shape) != self.shape:
            raise ValueError(f"pipeline prepared for shape {self.shape}, got {tuple(shape)}")

    def run_batch(self, frames, out=None, stream=None, out_dtype=np.float64):
        """Deblur a stack ``[N, H, W]``: CUDA tensor in -> CUDA tensor out (md_run), or host
        array in (uint8 camera frames, float32 or float64) -> host array out (float64 by
        default, float32 on request), copies pipelined inside the C ABI (md_run_host_ex)."""
        import torch
        if self._steps is not None:
            return self._run_batch_steps(frames, out, out_dtype)
        if isinstance(frames, torch.Tensor):
            self._check_shape(frames.shape[-2:])
            return self._plan.run(frames, out=out, stream=stream)
        a = np.asarray(frames)
        self._check_shape(a.shape[-2:])
        return self._plan.run_host(a, out=out, stream=stream, out_dtype=out_dtype)

    def _run_batch_steps(self, frames, out, out_dtype):
        import torch
        host = not isinstance(frames, torch.Tensor)
        t = _dev(np.asarray(frames, dtype=np.float64), self.dtype) if host else _dev(frames, self.dtype)
        self._check_shape(t.shape[-2:])
        u = self._run_steps(t)
        if not host:
            if out is not None:
                out.copy_(u)
                return out
            return u
        res = _host(u).astype(out_dtype, copy=False)
        if out is not None:
            out[...] = res
            return out
        return res

    def capture(self, batch: int = 1):
        """The pipeline for ``batch`` device-resident frames recorded as a CUDA graph
        (``plan.CapturedRun``): ``g(frames)`` copies the frames into the graph's input buffer and
        replays; the result is ``g.out``."""
        import torch
        if int(batch) < 1:
            raise ValueError("batch must be positive")
        if self._steps is not None:
            raise ValueError("a pipeline with a non-default divergence table runs step by step; capture needs "
                             "the default table")
        f = torch.zeros((int(batch),) + self.shape, dtype=torch_dtype(self.dtype), device="cuda")
        f.fill_(max(self.params.floor, 1.0))
        return self._plan.capture(f)

    def run_timed(self, f: Image) -> tuple[Image, StageTimes]:
        """Deconvolve one image with per-stage times from CUDA events on the launch stream
        (deconv.py:653-690). The per-iteration kernel path yields one time per iteration; the
        fused cluster kernel runs all iterations in one launch, whose time is split evenly."""
        import torch
        self._check_shape(f.shape)
        fd = _dev(f, self.dtype)
        if self._steps is not None:
            return self._run_timed_steps(fd)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        out, groups = self._plan.run_groups(fd)
        t1.record()
        torch.cuda.synchronize()
        wiener_ms = sum(ms for kind, ms in groups if kind == "init")
        iters = [ms for kind, ms in groups if kind == "iteration"]
        k = self.params.iterations
        if k and len(iters) != k:
            iters = [sum(iters) / k] * k
        total = max(t0.elapsed_time(t1), wiener_ms + sum(iters))
        return _image(out), StageTimes(wiener_ms=wiener_ms, iteration_ms=iters if k else [], total_ms=total)

    def _run_timed_steps(self, fd):
        import torch
        wplan, conv = self._steps
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(self.params.iterations + 2)]
        ev[0].record()
        u = wplan.run(fd)
        fpos = _clamp_dev(fd, self.params.floor)
        ev[1].record()
        for k in range(self.params.iterations):
            u = _iterate_steps(u, fpos, conv, self.params, self.lut)
            ev[k + 2].record()
        torch.cuda.synchronize()
        iters = [ev[k + 1].elapsed_time(ev[k + 2]) for k in range(self.params.iterations)]
        return _image(u), StageTimes(wiener_ms=ev[0].elapsed_time(ev[1]), iteration_ms=iters,
                                     total_ms=ev[0].elapsed_time(ev[-1]))

    def run(self, f: Image) -> Image:
        self._check_shape(f.shape)
        if self._steps is not None:
            return _image(self._run_steps(_dev(f, self.dtype)))
        return _image(self._plan.run(_dev(f, self.dtype)))


def wr3l(f: Image, h: Psf, params: DeconvParams, scenario: Scenario | None = None,
         dtype: str = "float64") -> Image:
    """Wiener filtering followed by RRRL iterations, one shot (deconv.py:696-703)."""
    return DeblurPipeline(f.shape, h, params, scenario, dtype=dtype).run(f)
