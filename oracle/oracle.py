"""TEST INFRASTRUCTURE — ctypes front-end for the FP64 CPU oracle.

Loads ``oracle/_build/libnlem_oracle.so`` (built from ``oracle/nlem_oracle.cpp``
by ``oracle/Makefile``).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline legs may import this module; the product path in
``paper_1501_03879_b200`` never does.

Each function restates one reference entry point (file:line cited in the C++).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libnlem_oracle.so")

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


class OracleParams(C.Structure):
    """Mirror of nlem::NlemParams (proj/include/nlem/nlem.hpp:23-35) + irls_tol."""

    _fields_ = [
        ("search", C.c_int32), ("patch", C.c_int32),
        ("h", C.c_double), ("sigma", C.c_double),
        ("solver", C.c_int32), ("solver_iters", C.c_int32),
        ("mu", C.c_double), ("epsilon", C.c_double),
        ("init_mode", C.c_int32), ("bounded", C.c_int32),
        ("lo", C.c_double), ("hi", C.c_double),
        ("threads", C.c_int32), ("irls_tol", C.c_double),
    ]


class OracleFailure(C.Structure):
    _fields_ = [("index", C.c_int64), ("iteration", C.c_int64), ("message", C.c_char * 256)]


class OracleError(Exception):
    def __init__(self, status: int, failure: OracleFailure | None = None):
        self.status = status
        self.index = failure.index if failure is not None else -1
        self.iteration = failure.iteration if failure is not None else 0
        msg = failure.message.decode() if failure is not None else ""
        super().__init__(msg or f"oracle status {status}")


def build() -> str:
    """Compile the oracle (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        srcs = ("nlem_oracle.cpp", "synth_oracle.cpp")
        if not os.path.exists(_SO) or any(
            os.path.getmtime(_SO) < os.path.getmtime(os.path.join(_HERE, f)) for f in srcs
        ):
            build()
        L = C.CDLL(_SO)
        L.oracle_mirror_index.restype = C.c_int64
        L.oracle_mirror_index.argtypes = [C.c_int64, C.c_int64]
        L.oracle_prox.argtypes = [_dp, _dp, C.c_int64, C.c_double, _dp]
        L.oracle_project_ball.argtypes = [_dp, C.c_int64, C.c_double, _dp]
        L.oracle_em_cost.restype = C.c_double
        L.oracle_em_cost.argtypes = [_dp, _dp, C.c_int64, C.c_int64, _dp]
        L.oracle_surrogate_cost.restype = C.c_double
        L.oracle_surrogate_cost.argtypes = [_dp, _dp, C.c_int64, C.c_int64, _dp, C.c_double]
        L.oracle_admm_batched.argtypes = [
            _dp, _dp, C.c_int64, C.c_int64, C.c_int64, _dp, C.c_int32, C.c_double, C.c_double,
            C.c_double, C.c_int64, C.c_double, _dp, _dp, _i64p, _dp, _dp, C.c_int32,
            C.POINTER(OracleFailure)]
        L.oracle_irls_batched.argtypes = [
            _dp, _dp, C.c_int64, C.c_int64, C.c_int64, _dp, C.c_double, C.c_int64, C.c_double,
            _dp, _dp, _i64p, _dp, C.c_int32, C.POINTER(OracleFailure)]
        L.oracle_build_patch_stack.argtypes = [
            _dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_double,
            _dp, _dp, _i64p, _i64p]
        L.oracle_patch_at.argtypes = [_dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32, _dp]
        L.oracle_patch_weights.argtypes = [_dp, C.c_int64, C.c_int64, C.c_int64, C.c_double, _dp]
        L.oracle_initial_patch.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_int32, _dp]
        L.oracle_nlem_denoise.argtypes = [
            _dp, C.c_int64, C.c_int64, OracleParams, C.c_int64, C.c_int64, _dp, _dp,
            C.POINTER(OracleFailure)]
        L.oracle_nlm_denoise.argtypes = [_dp, C.c_int64, C.c_int64, OracleParams, _dp]
        L.oracle_mse.restype = C.c_double
        L.oracle_mse.argtypes = [_dp, _dp, C.c_int64]
        L.oracle_psnr.restype = C.c_double
        L.oracle_psnr.argtypes = [_dp, _dp, C.c_int64]
        L.oracle_add_gaussian_noise.argtypes = [_dp, C.c_int64, C.c_double, C.c_uint64, _dp]
        L.oracle_optimality_residual.restype = C.c_double
        L.oracle_optimality_residual.argtypes = [
            _dp, _dp, C.c_int64, C.c_int64, C.c_int32, C.c_double, C.c_double, _dp]
        L.oracle_synth_noisy_image.argtypes = [
            C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_double, C.c_uint64, C.c_uint64,
            C.c_void_p, C.c_void_p]
        L.oracle_synth_point_sets.argtypes = [
            C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


def _check(status: int, failure: OracleFailure | None = None):
    if status != 0:
        raise OracleError(status, failure)


def mirror_index(i: int, n: int) -> int:
    return lib().oracle_mirror_index(i, n)


def prox_weighted_norm(v, u, lam):
    v, pv = _d(v)
    u, pu = _d(u)
    out = np.empty_like(v)
    _check(lib().oracle_prox(pv, pu, v.size, float(lam), out.ctypes.data_as(_dp)))
    return out


def project_ball(y, radius):
    y, py = _d(y)
    out = np.empty_like(y)
    _check(lib().oracle_project_ball(py, y.size, float(radius), out.ctypes.data_as(_dp)))
    return out


def em_cost(points, weights, x):
    points, pp = _d(points)
    weights, pw = _d(weights)
    x, px = _d(x)
    return lib().oracle_em_cost(pp, pw, points.shape[0], points.shape[1], px)


def surrogate_cost(points, weights, x, eps):
    points, pp = _d(points)
    weights, pw = _d(weights)
    x, px = _d(x)
    return lib().oracle_surrogate_cost(pp, pw, points.shape[0], points.shape[1], px, float(eps))


@dataclass
class SolveResult:
    minimizer: np.ndarray
    objective: np.ndarray
    iterations: np.ndarray
    trace_objective: np.ndarray | None = None
    trace_residual: np.ndarray | None = None


def admm_batched(points, weights, *, mu, max_iter, tol_primal=0.0, z_init=None, box=None,
                 trace=False, threads=0) -> SolveResult:
    """Batched proj/include/nlem/admm.hpp:26-86; points [B][n][d], weights [B][n]."""
    points, pp = _d(points)
    weights, pw = _d(weights)
    B, n, d = points.shape
    zi = None
    pzi = None
    if z_init is not None:
        zi, pzi = _d(np.broadcast_to(z_init, (B, d)))
    z = np.empty((B, d))
    obj = np.empty(B)
    it = np.empty(B, dtype=np.int64)
    to = tr = None
    if trace:
        to = np.full((B, max_iter), np.nan)
        tr = np.full((B, max_iter), np.nan)
    f = OracleFailure()
    bounded, lo, hi = (1, box[0], box[1]) if box is not None else (0, 0.0, 0.0)
    st = lib().oracle_admm_batched(
        pp, pw, B, n, d, pzi, bounded, lo, hi, float(mu), int(max_iter), float(tol_primal),
        z.ctypes.data_as(_dp), obj.ctypes.data_as(_dp), it.ctypes.data_as(_i64p),
        to.ctypes.data_as(_dp) if to is not None else None,
        tr.ctypes.data_as(_dp) if tr is not None else None, threads, C.byref(f))
    _check(st, f)
    return SolveResult(z, obj, it, to, tr)


def irls_batched(points, weights, *, epsilon, max_iter, tol=0.0, x_init=None, trace=False,
                 threads=0) -> SolveResult:
    """Batched proj/include/nlem/irls.hpp:21-68."""
    points, pp = _d(points)
    weights, pw = _d(weights)
    B, n, d = points.shape
    pxi = None
    if x_init is not None:
        xi, pxi = _d(np.broadcast_to(x_init, (B, d)))
    x = np.empty((B, d))
    obj = np.empty(B)
    it = np.empty(B, dtype=np.int64)
    to = np.full((B, max_iter), np.nan) if trace else None
    f = OracleFailure()
    st = lib().oracle_irls_batched(
        pp, pw, B, n, d, pxi, float(epsilon), int(max_iter), float(tol), x.ctypes.data_as(_dp),
        obj.ctypes.data_as(_dp), it.ctypes.data_as(_i64p),
        to.ctypes.data_as(_dp) if to is not None else None, threads, C.byref(f))
    _check(st, f)
    return SolveResult(x, obj, it, to, None)


def patch_at(img, row, col, k):
    img, pi = _d(img)
    out = np.empty(k * k)
    _check(lib().oracle_patch_at(pi, img.shape[0], img.shape[1], row, col, k, out.ctypes.data_as(_dp)))
    return out


def patch_weights(patches, center, h):
    patches, pp = _d(patches)
    w = np.empty(patches.shape[0])
    _check(lib().oracle_patch_weights(pp, patches.shape[0], patches.shape[1], center, float(h),
                                      w.ctypes.data_as(_dp)))
    return w


def build_patch_stack(img, row, col, search, k, h):
    """proj/src/patch.cpp:90-114 -> (patches [n][d], weights [n], self_column)."""
    img, pi = _d(img)
    patches = np.empty((search * search, k * k))
    w = np.empty(search * search)
    n = C.c_int64()
    sc = C.c_int64()
    _check(lib().oracle_build_patch_stack(pi, img.shape[0], img.shape[1], row, col, search, k,
                                          float(h), patches.ctypes.data_as(_dp),
                                          w.ctypes.data_as(_dp), C.byref(n), C.byref(sc)))
    return patches[: n.value].copy(), w[: n.value].copy(), sc.value


def initial_patch(patches, weights, self_col, mode):
    patches, pp = _d(patches)
    weights, pw = _d(weights)
    out = np.empty(patches.shape[1])
    _check(lib().oracle_initial_patch(pp, pw, patches.shape[0], patches.shape[1], self_col, mode,
                                      out.ctypes.data_as(_dp)))
    return out


SOLVERS = {"admm": 0, "irls": 1, "nlm": 2}
INITS = {"noisy": 0, "nlm": 1}


def make_params(*, search=21, patch=7, h, sigma=0.0, solver="admm", solver_iters=4, mu=1e-3,
                epsilon=1e-6, init_mode="noisy", box=(0.0, 255.0), threads=0, irls_tol=0.0):
    p = OracleParams()
    p.search, p.patch, p.h, p.sigma = search, patch, float(h), float(sigma)
    p.solver, p.solver_iters = SOLVERS[solver], solver_iters
    p.mu, p.epsilon = float(mu), float(epsilon)
    p.init_mode = INITS[init_mode]
    if box is None:
        p.bounded, p.lo, p.hi = 0, 0.0, 0.0
    else:
        p.bounded, p.lo, p.hi = 1, float(box[0]), float(box[1])
    p.threads = threads
    p.irls_tol = float(irls_tol)
    return p


def nlem_denoise(noisy, params: OracleParams, *, rows=None, snapshots=False):
    """proj/src/nlem.cpp:68-90 (and :92-128 with snapshots=True).

    rows=(r0, r1) restricts the computed output rows (others stay NaN).
    Returns out, or (out, frames) with snapshots.
    """
    noisy, pn = _d(noisy)
    H, W = noisy.shape
    r0, r1 = rows if rows is not None else (0, H)
    out = np.full((H, W), np.nan)
    frames = np.full((params.solver_iters, H, W), np.nan) if snapshots else None
    f = OracleFailure()
    st = lib().oracle_nlem_denoise(pn, H, W, params, r0, r1, out.ctypes.data_as(_dp),
                                   frames.ctypes.data_as(_dp) if frames is not None else None,
                                   C.byref(f))
    _check(st, f)
    return (out, frames) if snapshots else out


def nlm_denoise(noisy, params: OracleParams):
    noisy, pn = _d(noisy)
    out = np.empty_like(noisy)
    _check(lib().oracle_nlm_denoise(pn, noisy.shape[0], noisy.shape[1], params,
                                    out.ctypes.data_as(_dp)))
    return out


def psnr(a, b):
    a, pa = _d(a)
    b, pb = _d(b)
    return lib().oracle_psnr(pa, pb, a.size)


def mse(a, b):
    a, pa = _d(a)
    b, pb = _d(b)
    return lib().oracle_mse(pa, pb, a.size)


def add_gaussian_noise(clean, sigma, seed):
    clean, pc = _d(clean)
    out = np.empty_like(clean)
    lib().oracle_add_gaussian_noise(pc, clean.size, float(sigma), int(seed), out.ctypes.data_as(_dp))
    return out


def optimality_residual(points, weights, z, box=None):
    points, pp = _d(points)
    weights, pw = _d(weights)
    z, pz = _d(z)
    bounded, lo, hi = (1, box[0], box[1]) if box is not None else (0, 0.0, 0.0)
    return lib().oracle_optimality_residual(pp, pw, points.shape[0], points.shape[1], bounded,
                                            lo, hi, pz)


# ---- seeded inputs, independent of the product library (oracle/synth_oracle.cpp)
SYNTH_CONFIGS = {
    0: dict(rows=128, cols=128, rects=12, disks=8, sigma=20.0),
    2: dict(rows=512, cols=512, rects=40, disks=30, sigma=20.0),
    3: dict(rows=4096, cols=4096, rects=2000, disks=1500, sigma=30.0),
}


def synth_noisy_image(rows, cols, rects, disks, sigma, image_seed=0, noise_seed=1):
    """(clean, noisy) float32 images of the BASELINE.json generator."""
    clean = np.empty((rows, cols), np.float32)
    noisy = np.empty((rows, cols), np.float32)
    lib().oracle_synth_noisy_image(rows, cols, rects, disks, float(sigma), image_seed, noise_seed,
                                   clean.ctypes.data, noisy.ctypes.data)
    return clean, noisy


def synth_config_image(cfg: int, **over):
    c = dict(SYNTH_CONFIGS[cfg])
    c.update(over)
    return synth_noisy_image(c["rows"], c["cols"], c["rects"], c["disks"], c["sigma"])


def synth_point_sets(batch, n=441, d=49, seed_base=1000, first=0):
    """Config-1 point sets: (points [B][n][d], weights [B][n]) float32."""
    pts = np.empty((batch, n, d), np.float32)
    w = np.empty((batch, n), np.float32)
    lib().oracle_synth_point_sets(batch, n, d, seed_base, first, pts.ctypes.data, w.ctypes.data)
    return pts, w
