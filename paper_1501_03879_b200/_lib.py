"""ctypes binding of the C-ABI in include/nlem_b200.h (libnlem_b200.so, sm_100a).

The library is built in-tree by ``paper_1501_03879_b200.build``.  There is no
CPU fallback: if the shared object is missing or cannot be loaded, importing
the compute API raises.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

SO_PATH = _build.SO

_fp = C.POINTER(C.c_float)
_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)

NLEM_OK, NLEM_INVALID_ARGUMENT, NLEM_NUMERIC_FAILURE, NLEM_CUDA_ERROR = 0, 1, 2, 3
SOLVER_ADMM, SOLVER_IRLS, SOLVER_NLM_ONLY = 0, 1, 2
INIT_NOISY_PATCH, INIT_NLM_PATCH = 0, 1


class Failure(C.Structure):
    _fields_ = [("index", C.c_int64), ("iteration", C.c_int64), ("kind", C.c_int32),
                ("message", C.c_char * 256)]


class Box(C.Structure):
    _fields_ = [("bounded", C.c_int32), ("lower", C.c_float), ("upper", C.c_float)]


class AdmmConfigC(C.Structure):
    _fields_ = [("mu", C.c_float), ("max_iter", C.c_int32), ("tol_primal", C.c_float)]


class IrlsConfigC(C.Structure):
    _fields_ = [("epsilon", C.c_float), ("max_iter", C.c_int32), ("tol", C.c_float)]


class ParamsC(C.Structure):
    _fields_ = [("search", C.c_int32), ("patch", C.c_int32), ("h", C.c_float),
                ("sigma", C.c_float), ("solver", C.c_int32), ("solver_iters", C.c_int32),
                ("mu", C.c_float), ("epsilon", C.c_float), ("init_mode", C.c_int32),
                ("range", Box), ("irls_tol", C.c_float)]


# Every symbol include/nlem_b200.h declares (checked by tests/test_abi_cpu.py).
EXPORTS = [
    "nlem_version", "nlem_status_string", "nlem_validate_params", "nlem_default_init_mode",
    "nlem_admm_batched", "nlem_admm_batched_host", "nlem_irls_batched",
    "nlem_irls_batched_host", "nlem_denoise",
    "nlem_denoise_rows", "nlem_denoise_rows_host", "nlem_denoise_host", "nlem_denoise_multi_host",
    "nlm_denoise", "nlem_band_halo",
    "nlem_add_gaussian_noise", "nlem_synth_clean_image", "nlem_synth_noisy_image",
    "nlem_synth_point_sets", "nlem_frames_psnr", "nlem_optimality_residual_batched",
    "nlem_patch_stack_host", "nlem_solve_patch_host",
]

_lib = None


def load(build_if_missing: bool = True):
    """Load (building first if needed) the in-tree shared library."""
    global _lib
    if _lib is not None:
        return _lib
    so_path = SO_PATH
    variant = os.environ.get("NLEM_LIB_VARIANT", "")  # A/B builds (build.py --variant=...)
    if variant:
        so_path = _build.variant_path(variant)
    elif build_if_missing:
        _build.build()
    if not os.path.exists(so_path):
        raise RuntimeError(f"NLEM CUDA library missing: {so_path} (run paper_1501_03879_b200.build)")
    L = C.CDLL(so_path)
    vp = C.c_void_p
    L.nlem_version.restype = C.c_char_p
    L.nlem_status_string.restype = C.c_char_p
    L.nlem_status_string.argtypes = [C.c_int]
    L.nlem_validate_params.argtypes = [C.POINTER(ParamsC), C.POINTER(Failure)]
    L.nlem_default_init_mode.restype = C.c_int32
    L.nlem_default_init_mode.argtypes = [C.c_float]
    L.nlem_band_halo.restype = C.c_int64
    L.nlem_band_halo.argtypes = [C.POINTER(ParamsC)]
    L.nlem_admm_batched.argtypes = [vp, vp, C.c_int64, C.c_int64, C.c_int64, vp, Box, AdmmConfigC,
                                    vp, vp, vp, vp, vp, C.POINTER(Failure), vp]
    L.nlem_admm_batched_host.argtypes = [vp, vp, C.c_int64, C.c_int64, C.c_int64, vp, Box,
                                         AdmmConfigC, vp, vp, vp, vp, vp, C.POINTER(Failure),
                                         C.c_int32]
    L.nlem_irls_batched.argtypes = [vp, vp, C.c_int64, C.c_int64, C.c_int64, vp, IrlsConfigC, vp,
                                    vp, vp, vp, C.POINTER(Failure), vp]
    L.nlem_irls_batched_host.argtypes = [vp, vp, C.c_int64, C.c_int64, C.c_int64, vp, IrlsConfigC,
                                         vp, vp, vp, vp, C.POINTER(Failure), C.c_int32]
    L.nlem_denoise.argtypes = [vp, C.c_int64, C.c_int64, C.POINTER(ParamsC), vp, vp,
                               C.POINTER(Failure), vp]
    L.nlem_denoise_rows.argtypes = [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                    C.c_int64, C.POINTER(ParamsC), vp, vp, C.POINTER(Failure), vp]
    L.nlem_denoise_rows_host.argtypes = [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                         C.c_int64, C.c_int64, C.POINTER(ParamsC), vp, vp,
                                         C.POINTER(Failure), C.c_int32]
    L.nlem_denoise_host.argtypes = [vp, C.c_int64, C.c_int64, C.POINTER(ParamsC), vp, vp,
                                    C.POINTER(Failure), C.c_int32]
    L.nlem_denoise_multi_host.argtypes = [vp, C.c_int64, C.c_int64, C.POINTER(ParamsC), vp, vp,
                                          C.POINTER(C.c_int32), C.c_int32, C.POINTER(Failure)]
    L.nlm_denoise.argtypes = [vp, C.c_int64, C.c_int64, C.POINTER(ParamsC), vp,
                              C.POINTER(Failure), vp]
    L.nlem_frames_psnr.argtypes = [vp, vp, C.c_int64, C.c_int64, vp, C.POINTER(Failure), vp]
    L.nlem_optimality_residual_batched.argtypes = [vp, vp, C.c_int64, C.c_int64, C.c_int64, Box, vp,
                                                   vp, C.POINTER(Failure), vp]
    L.nlem_patch_stack_host.argtypes = [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                        C.c_int32, C.c_float, vp, vp, C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int64), C.POINTER(Failure), C.c_int32]
    L.nlem_solve_patch_host.argtypes = [vp, vp, C.c_int64, C.c_int64, C.c_int64, C.POINTER(ParamsC),
                                        vp, vp, C.POINTER(Failure), C.c_int32]
    L.nlem_add_gaussian_noise.argtypes = [vp, C.c_int64, C.c_double, C.c_uint64, vp]
    L.nlem_synth_clean_image.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_uint64, vp]
    L.nlem_synth_noisy_image.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_double,
                                         C.c_uint64, C.c_uint64, vp, vp]
    L.nlem_synth_point_sets.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int64, vp,
                                        vp, C.c_int32]
    _lib = L
    return L
