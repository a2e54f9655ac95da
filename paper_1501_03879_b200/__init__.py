"""B200-native (sm_100a) NLEM / EM-ADMM hot path.

The product is the C-ABI library ``_lib/libnlem_b200.so`` (include/nlem_b200.h);
this package is its Python front-end mirroring the reference API
(proj/include/nlem/*.hpp).  No CPU fallback exists: compute calls raise when
the CUDA library or a GPU is missing.
"""
from .api import (  # noqa: F401
    AdmmConfig, BoxConstraint, CudaError, InvalidArgument, IrlsConfig, NlemParams,
    NumericFailure, PatchSolve, PatchStack, SolverResult, TraceRecord, admm_euclidean_median,
    band_halo, build_patch_stack, solve_patch,
    default_init_mode, frames_psnr, optimality_residual, irls_euclidean_median, nlem_denoise, nlem_denoise_host,
    nlem_denoise_multi_host,
    nlem_denoise_rows, nlem_denoise_rows_host, nlem_denoise_snapshots, nlm_denoise, validate,
)
