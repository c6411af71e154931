"""Device plan: the host-side owner of one ``md_plan`` (include/mdcuda.h).

A ``GpuPlan`` fixes the frame shape, the PSF, the parameters, the convolver realisation and
the arithmetic type, and keeps the device tables the CUDA library builds for them (taps,
twiddles, Wiener multiplier, divergence table, scratch). It is the counterpart of the
precomputation in ``DeblurPipeline.__init__`` (deconv.py:611-643) and ``make_convolver``
(deconv.py:379-403). Tensors passed in are torch CUDA tensors (torch is only the device
memory / stream plumbing); numpy arrays are staged through the device by the callers.
"""

from __future__ import annotations

import contextlib
import ctypes

import numpy as np

from . import _lib as L
from .core import BlurAxis, DeconvParams, Psf, PsfKind

_DTYPES = {"float64": L.MD_F64, "float32": L.MD_F32}
_CONV = {"box": L.MD_CONV_BOX, "spatial": L.MD_CONV_SPATIAL, "fourier": L.MD_CONV_FOURIER,
         "fourier2d": L.MD_CONV_FOURIER2D}


def torch_dtype(dtype: str):
    import torch
    return {"float64": torch.float64, "float32": torch.float32}[dtype]


def _stream_ptr(stream) -> int | None:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream or None


class GpuPlan:
    """One compiled problem (shape x PSF x params x convolver x dtype) on the device."""

    def __init__(self, shape, psf: Psf, params: DeconvParams, conv: str, init: str = "wiener",
                 dtype: str = "float64", rl: bool = False, force_fft2d: bool = False,
                 fused: bool | None = None, generic_lines: bool = False, big_fft: bool = False):
        if dtype not in _DTYPES:
            raise ValueError(f"dtype must be one of {sorted(_DTYPES)}")
        if conv not in _CONV:
            raise ValueError(f"unknown convolver mode {conv!r}")
        self.lib = L.lib()
        self.shape = (int(shape[0]), int(shape[1]))
        self.psf, self.params, self.conv, self.dtype = psf, params, conv, dtype
        w = np.ascontiguousarray(psf.weights, dtype=np.float64)
        self._w = w                                # keep alive during plan creation
        d = L.PlanDesc()
        d.height, d.width = self.shape
        d.dtype = _DTYPES[dtype]
        if psf.kind is PsfKind.GENERAL_2D:
            d.psf_kind = L.MD_PSF_GENERAL_2D
            d.psf_axis = L.MD_AXIS_NONE
            d.psf_rows, d.psf_cols = w.shape
            d.center_row, d.center_col = psf.center
        else:
            d.psf_kind = L.MD_PSF_BOX_1D if psf.kind is PsfKind.UNIFORM_BOX_1D else L.MD_PSF_GENERAL_1D
            d.psf_axis = L.MD_AXIS_VERTICAL if psf.axis is BlurAxis.VERTICAL else L.MD_AXIS_HORIZONTAL
            d.psf_rows, d.psf_cols = w.shape[0], 1
            d.center_row, d.center_col = int(psf.center), 0
            d.box_length = float(psf.length) if psf.length is not None else 0.0
        d.psf_weights = w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        d.conv = _CONV[conv]
        d.init = L.MD_INIT_WIENER if init == "wiener" else L.MD_INIT_CLAMPED
        d.iterations = int(params.iterations)
        d.flags = ((L.MD_FLAG_RL if rl else 0) | (L.MD_FLAG_FORCE_FFT2D if force_fft2d else 0)
                   | (L.MD_FLAG_GENERIC_LINES if generic_lines else 0) | (L.MD_FLAG_BIG_FFT if big_fft else 0))
        d.wiener_k, d.alpha = params.wiener_k, (0.0 if rl else params.alpha)
        d.eps_data, d.eps_reg, d.floor = params.eps_data, params.eps_reg, params.floor
        h = ctypes.c_void_p()
        L.check(self.lib.md_plan_create(ctypes.byref(d), ctypes.byref(h)))
        self._h = h
        if fused is not None:
            L.check(self.lib.md_plan_set_fused(h, 1 if fused else 0))

    # ------------------------------------------------------------------ lifecycle
    def close(self) -> None:
        if getattr(self, "_h", None):
            self.lib.md_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def describe(self) -> str:
        return self.lib.md_plan_describe(self._h).decode()

    @property
    def fused(self) -> bool:
        return bool(self.lib.md_plan_is_fused(self._h))

    def fused_geometry(self) -> dict:
        """The 1D cluster kernel's launch shape: CTAs per cluster, co-resident clusters, CTAs per
        SM and the SMs they keep busy (zeros when the plan does not use it)."""
        c, r, p = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        L.check(self.lib.md_plan_fused_geometry(self._h, ctypes.byref(c), ctypes.byref(r), ctypes.byref(p)))
        busy = -(-(c.value * r.value) // p.value) if p.value else 0
        return {"cluster_ctas": c.value, "resident_clusters": r.value, "ctas_per_sm": p.value, "sms_busy": busy}

    def set_fused(self, on: bool) -> None:
        L.check(self.lib.md_plan_set_fused(self._h, 1 if on else 0))

    def set_chunk(self, frames: int) -> None:
        L.check(self.lib.md_plan_set_chunk(self._h, int(frames)))

    def launch_count(self, batch: int) -> int:
        return int(self.lib.md_run_launch_count(self._h, int(batch)))

    # ------------------------------------------------------------------ helpers
    def _check_frames(self, t, name="f"):
        import torch
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise TypeError(f"{name} must be a CUDA tensor")
        if t.dtype != torch_dtype(self.dtype):
            raise TypeError(f"{name} must have dtype {self.dtype}, got {t.dtype}")
        if tuple(t.shape[-2:]) != self.shape:
            raise ValueError(f"plan prepared for shape {self.shape}, got {tuple(t.shape[-2:])}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        return 1 if t.dim() == 2 else int(np.prod(t.shape[:-2]))

    def empty_like(self, t):
        import torch
        return torch.empty_like(t, memory_format=torch.contiguous_format)

    # ------------------------------------------------------------------ entry points
    def run(self, f, out=None, stream=None):
        """Whole pipeline on device frames ``[..., H, W]`` (md_run)."""
        n = self._check_frames(f)
        out = self.empty_like(f) if out is None else out
        self._check_frames(out, "out")
        L.check(self.lib.md_run(self._h, f.data_ptr(), out.data_ptr(), n, _stream_ptr(stream)))
        return out

    def capture(self, f, out=None) -> "CapturedRun":
        """Record ``run(f, out)`` into a CUDA graph for fixed device buffers (video-rate use: one
        graph launch per batch instead of one host call per kernel). Runs once uncaptured first,
        which sizes the plan's scratch; afterwards write new frames into ``f`` and ``replay()``."""
        import torch
        self._check_frames(f)
        out = self.empty_like(f) if out is None else out
        self._check_frames(out, "out")
        side = torch.cuda.Stream(device=f.device)
        side.wait_stream(torch.cuda.current_stream(f.device))
        with torch.cuda.stream(side):
            self.run(f, out, stream=side)
        graph = torch.cuda.CUDAGraph()
        # relaxed: the launchers set kernel attributes (cudaFuncSetAttribute) while enqueuing
        with torch.cuda.graph(graph, stream=side, capture_error_mode="relaxed"):
            self.run(f, out, stream=side)
        torch.cuda.current_stream(f.device).wait_stream(side)
        return CapturedRun(self, graph, f, out)

    def run_profile(self, f, out=None, stream=None) -> dict:
        """md_run with CUDA events per launch group: {"init_ms", "iter_ms", "layout_ms", "groups"}."""
        n = self._check_frames(f)
        out = self.empty_like(f) if out is None else out
        ms = (ctypes.c_double * 4)()
        L.check(self.lib.md_run_profile(self._h, f.data_ptr(), out.data_ptr(), n, _stream_ptr(stream), ms))
        return {"init_ms": ms[0], "iter_ms": ms[1], "layout_ms": ms[2], "groups": int(ms[3])}

    def run_groups(self, f, out=None, stream=None):
        """md_run with one CUDA event per launch group -> (out, [(kind, ms), ...])."""
        n = self._check_frames(f)
        out = self.empty_like(f) if out is None else out
        cap = 4096
        ms = (ctypes.c_double * cap)()
        kinds = (ctypes.c_int32 * cap)()
        cnt = ctypes.c_int32()
        L.check(self.lib.md_run_profile_groups(self._h, f.data_ptr(), out.data_ptr(), n, _stream_ptr(stream), ms,
                                               kinds, cap, ctypes.byref(cnt)))
        names = {0: "init", 1: "iteration", 2: "layout"}
        return out, [(names[kinds[i]], ms[i]) for i in range(cnt.value)]

    _IO = {np.dtype(np.float64): L.MD_IO_F64, np.dtype(np.float32): L.MD_IO_F32, np.dtype(np.uint8): L.MD_IO_U8}

    def run_host(self, f: np.ndarray, out: np.ndarray | None = None, stream=None,
                 out_dtype=np.float64) -> np.ndarray:
        """Whole pipeline from HOST frames (uint8 / float32 / float64) to HOST results
        (float32 / float64), copies pipelined inside the C ABI (md_run_host_ex). Pinned
        (page-locked) buffers make the copies asynchronous."""
        f = np.asarray(f)
        if f.dtype not in self._IO:
            f = f.astype(np.float64)
        f = np.ascontiguousarray(f)
        if f.shape[-2:] != self.shape:
            raise ValueError(f"plan prepared for shape {self.shape}, got {f.shape[-2:]}")
        n = 1 if f.ndim == 2 else int(np.prod(f.shape[:-2]))
        out = np.empty(f.shape, dtype=out_dtype) if out is None else out
        if out.dtype not in (np.float32, np.float64, np.uint8) or out.shape != f.shape or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float32/float64/uint8 array of the input's shape "
                             "(uint8: write_pgm quantisation)")
        L.check(self.lib.md_run_host_ex(self._h, f.ctypes.data, self._IO[f.dtype], out.ctypes.data,
                                        self._IO[out.dtype], n, _stream_ptr(stream)))
        return out

    def wiener(self, f, out=None, stream=None):
        n = self._check_frames(f)
        out = self.empty_like(f) if out is None else out
        L.check(self.lib.md_wiener(self._h, f.data_ptr(), out.data_ptr(), n, _stream_ptr(stream)))
        return out

    def convolve(self, a, which: int, out=None, stream=None):
        n = self._check_frames(a, "a")
        out = self.empty_like(a) if out is None else out
        L.check(self.lib.md_convolve(self._h, a.data_ptr(), out.data_ptr(), n, which, _stream_ptr(stream)))
        return out

    def adjoint_pair(self, p, q, stream=None):
        n = self._check_frames(p, "p")
        self._check_frames(q, "q")
        op, oq = self.empty_like(p), self.empty_like(q)
        L.check(self.lib.md_adjoint_pair(self._h, p.data_ptr(), q.data_ptr(), op.data_ptr(), oq.data_ptr(),
                                         n, _stream_ptr(stream)))
        return op, oq

    def rrrl_step(self, u, f, b, w=None, d=None, alpha: float = 0.0, stream=None):
        n = self._check_frames(u, "u")
        out = self.empty_like(u)
        L.check(self.lib.md_rrrl_step(self._h, u.data_ptr(), f.data_ptr(), b.data_ptr(),
                                      None if w is None else w.data_ptr(),
                                      None if d is None else d.data_ptr(),
                                      out.data_ptr(), n, float(alpha), _stream_ptr(stream)))
        return out


class CapturedRun:
    """A ``GpuPlan.run`` recorded as a CUDA graph over fixed buffers ``f`` -> ``out``. The
    graph holds the plan's device pointers: keep the plan alive and do not use it from another
    stream while a replay may be running (replays are ordered only by their own stream)."""

    def __init__(self, plan: GpuPlan, graph, f, out):
        self.plan, self.graph, self.f, self.out = plan, graph, f, out

    def replay(self, stream=None):
        """Launch the recorded pipeline on ``stream`` (default: the current stream); returns
        ``out``."""
        import torch
        if stream is None:
            self.graph.replay()
        else:
            with torch.cuda.stream(stream):
                self.graph.replay()
        return self.out

    def __call__(self, frames=None, stream=None):
        """Copy ``frames`` (a device tensor of ``f``'s shape) into the input buffer, replay."""
        if frames is not None:
            import torch
            with torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext():
                self.f.copy_(frames, non_blocking=True)
        return self.replay(stream)


def dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float64:
        return L.MD_F64
    if t.dtype == torch.float32:
        return L.MD_F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def device_min(t, stream=None) -> float:
    out = ctypes.c_double()
    L.check(L.lib().md_min(dtype_code(t), t.data_ptr(), t.numel(), ctypes.byref(out), _stream_ptr(stream)))
    return out.value


def convert_dev(src, dst, stream=None):
    """Element type conversion of device tensors (uint8 / float32 / float64 -> float32 / float64,
    float -> uint8 with write_pgm quantisation) by the library's conversion kernel (md_convert),
    on `stream`, without synchronising."""
    import torch
    io = {torch.float64: L.MD_IO_F64, torch.float32: L.MD_IO_F32, torch.uint8: L.MD_IO_U8}
    if src.numel() != dst.numel() or not src.is_contiguous() or not dst.is_contiguous():
        raise ValueError("convert_dev needs contiguous tensors of equal size")
    if src.dtype not in io or dst.dtype not in io or (dst.dtype == torch.uint8 and src.dtype == torch.uint8):
        raise TypeError(f"unsupported conversion {src.dtype} -> {dst.dtype}")
    L.check(L.lib().md_convert(src.data_ptr(), io[src.dtype], dst.data_ptr(), io[dst.dtype], src.numel(),
                               _stream_ptr(stream)))
    return dst


def guard_(t, stream=None):
    L.check(L.lib().md_guard(dtype_code(t), t.data_ptr(), t.numel(), _stream_ptr(stream)))
    return t


def robust_weight_dev(f, b, eps_data: float, floor: float, assume_floored: bool = False, stream=None):
    out = b.new_empty(b.shape)
    L.check(L.lib().md_robust_weight(dtype_code(f), f.data_ptr(), b.data_ptr(), out.data_ptr(), f.numel(),
                                     eps_data, floor, 1 if assume_floored else 0, _stream_ptr(stream)))
    return out


def diffusion_dev(u, eps_reg: float, stream=None):
    out = u.new_empty(u.shape)
    h, w = u.shape[-2:]
    n = 1 if u.dim() == 2 else int(np.prod(u.shape[:-2]))
    L.check(L.lib().md_diffusion(dtype_code(u), u.data_ptr(), out.data_ptr(), n, h, w, eps_reg,
                                 _stream_ptr(stream)))
    return out
