"""ctypes binding of the in-tree CUDA library (``libmdcuda.so``, C ABI in include/mdcuda.h).

There is no CPU fallback: if the library or a CUDA device is missing, every compute call
raises immediately (``CudaUnavailable``). Status codes map to the reference's exception
types (ValueError, ContractError -- core.py:39-40 -- MemoryError, RuntimeError).
"""

from __future__ import annotations

import ctypes
import os

from .core import ContractError

_HERE = os.path.dirname(os.path.abspath(__file__))
# MD_LIB: an alternative build of the same library (kernel experiments, scripts/build_variant.py)
LIB_PATH = os.environ.get("MD_LIB") or os.path.join(_HERE, "libmdcuda.so")

MD_OK, MD_EINVAL, MD_ECONTRACT, MD_ECUDA, MD_ENOMEM = 0, -1, -2, -3, -4
MD_F64, MD_F32 = 0, 1
MD_PSF_GENERAL_2D, MD_PSF_GENERAL_1D, MD_PSF_BOX_1D = 0, 1, 2
MD_AXIS_NONE, MD_AXIS_VERTICAL, MD_AXIS_HORIZONTAL = -1, 0, 1
MD_CONV_BOX, MD_CONV_SPATIAL, MD_CONV_FOURIER, MD_CONV_FOURIER2D = 0, 1, 2, 3
MD_INIT_WIENER, MD_INIT_CLAMPED = 0, 1
MD_IO_F64, MD_IO_F32, MD_IO_U8 = 0, 1, 2
MD_FLAG_RL, MD_FLAG_NO_FUSED, MD_FLAG_FORCE_FFT2D, MD_FLAG_GENERIC_LINES, MD_FLAG_BIG_FFT = 1, 2, 4, 8, 16


class CudaUnavailable(RuntimeError):
    """The CUDA library or device is missing; there is deliberately no fallback."""


class PlanDesc(ctypes.Structure):
    """Mirror of ``md_plan_desc`` (include/mdcuda.h)."""

    _fields_ = [
        ("height", ctypes.c_int32), ("width", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("psf_kind", ctypes.c_int32), ("psf_axis", ctypes.c_int32),
        ("psf_rows", ctypes.c_int32), ("psf_cols", ctypes.c_int32),
        ("center_row", ctypes.c_int32), ("center_col", ctypes.c_int32),
        ("box_length", ctypes.c_double),
        ("psf_weights", ctypes.POINTER(ctypes.c_double)),
        ("conv", ctypes.c_int32), ("init", ctypes.c_int32),
        ("iterations", ctypes.c_int32), ("flags", ctypes.c_uint32),
        ("wiener_k", ctypes.c_double), ("alpha", ctypes.c_double),
        ("eps_data", ctypes.c_double), ("eps_reg", ctypes.c_double), ("floor", ctypes.c_double),
    ]


_P = ctypes.c_void_p
_I32, _I64, _D = ctypes.c_int32, ctypes.c_int64, ctypes.c_double

# name -> (restype, argtypes); every symbol include/mdcuda.h declares
SIGNATURES = {
    "md_abi_version": (_I32, []),
    "md_last_error": (ctypes.c_char_p, []),
    "md_device_sm_count": (_I32, []),
    "md_plan_create": (_I32, [ctypes.POINTER(PlanDesc), ctypes.POINTER(_P)]),
    "md_plan_destroy": (_I32, [_P]),
    "md_plan_scratch_bytes": (_I64, [_P, _I64]),
    "md_plan_describe": (ctypes.c_char_p, [_P]),
    "md_plan_set_chunk": (_I32, [_P, _I64]),
    "md_plan_set_fused": (_I32, [_P, _I32]),
    "md_plan_is_fused": (_I32, [_P]),
    "md_plan_fused_geometry": (_I32, [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "md_run": (_I32, [_P, _P, _P, _I64, _P]),
    "md_run_host": (_I32, [_P, _P, _P, _I64, _P]),
    "md_run_host_ex": (_I32, [_P, _P, _I32, _P, _I32, _I64, _P]),
    "md_convert": (_I32, [_P, _I32, _P, _I32, _I64, _P]),
    "md_run_launch_count": (_I32, [_P, _I64]),
    "md_run_profile": (_I32, [_P, _P, _P, _I64, _P, ctypes.POINTER(_D)]),
    "md_run_profile_groups": (_I32, [_P, _P, _P, _I64, _P, ctypes.POINTER(_D), ctypes.POINTER(_I32), _I32,
                                     ctypes.POINTER(_I32)]),
    "md_wiener": (_I32, [_P, _P, _P, _I64, _P]),
    "md_convolve": (_I32, [_P, _P, _P, _I64, _I32, _P]),
    "md_adjoint_pair": (_I32, [_P, _P, _P, _P, _P, _I64, _P]),
    "md_robust_weight": (_I32, [_I32, _P, _P, _P, _I64, _D, _D, _I32, _P]),
    "md_diffusion": (_I32, [_I32, _P, _P, _I64, _I32, _I32, _D, _P]),
    "md_rrrl_step": (_I32, [_P, _P, _P, _P, _P, _P, _P, _I64, _D, _P]),
    "md_guard": (_I32, [_I32, _P, _I64, _P]),
    "md_lut_build": (_I32, [_P, _I64, _D, _D, _P]),
    "md_lut_r1_custom": (_I32, [_P, _I64, _D, _D, _D, _D, _D, _D, _P, _P, _I64, _P]),
    "md_robust_weight_custom": (_I32, [_I32, _P, _I64, _D, _D, _D, _D, _D, _D, _P, _P, _P, _I64, _D, _D, _I32, _P]),
    "md_clamp": (_I32, [_I32, _P, _P, _I64, _D, _P]),
    "md_ratio": (_I32, [_I32, _P, _P, _P, _P, _I64, _P]),
    "md_combine": (_I32, [_I32, _P, _P, _P, _P, _P, _I64, _D, _P]),
    "md_lut_r1": (_I32, [_I32, _P, _P, _I64, _P]),
    "md_lut_table": (_I32, [ctypes.POINTER(_D), _I64]),
    "md_min": (_I32, [_I32, _P, _I64, ctypes.POINTER(_D), _P]),
    "md_fft": (_I32, [_I32, _P, _I32, _I64, _I32, _P]),
    "md_slab_halo": (_I32, [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "md_slab_prepare": (_I32, [_P, _I32, _I32, ctypes.POINTER(_P)]),
    "md_slab_rows_fft": (_I32, [_P, _P, _P, _I32, _I32, _D, _P]),
    "md_slab_cols_filter": (_I32, [_P, _P, _I32, _P, _P]),
    "md_slab_wiener_epilogue": (_I32, [_P, _P, _P, _P, _P, _I32, _P]),
    "md_slab_iterate": (_I32, [_P, _P, _P, _P, _P, _P, _I32, _I32, _P]),
    "md_slab_stage": (_I32, [_P, _P, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _I32, _I32, _P]),
    "md_slab_bands": (_I32, [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32), ctypes.POINTER(_I32),
                             ctypes.POINTER(_I32)]),
}

_lib = None


def load_library() -> ctypes.CDLL:
    """Load libmdcuda.so (no device needed). Raises CudaUnavailable if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaUnavailable(
                f"{LIB_PATH} is missing: build it with `python -m paper_1212_2245_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def lib() -> ctypes.CDLL:
    """The library, after checking that a CUDA device is present (fails loudly otherwise)."""
    L = load_library()
    import torch
    if not torch.cuda.is_available():
        raise CudaUnavailable("no CUDA device: the deblurring kernels need a B200 (sm_100a); "
                              "there is no CPU fallback")
    return L


def check(rc: int) -> None:
    if rc == MD_OK:
        return
    msg = load_library().md_last_error().decode(errors="replace")
    if rc == MD_EINVAL:
        raise ValueError(msg)
    if rc == MD_ECONTRACT:
        raise ContractError(msg)
    if rc == MD_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"CUDA failure: {msg}")
