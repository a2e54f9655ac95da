"""Python mirror of the reference's public API for the NLEM / EM-ADMM path.

Same names, argument meaning and error behaviour as the reference's C++ entry
points (proj/include/nlem/{types,admm,irls,nlem}.hpp); every call runs on the
GPU through the C-ABI (include/nlem_b200.h).  Inputs may be torch CUDA tensors
(device path, enqueued on the current stream) or numpy / host arrays (copied
through the library's ``*_host`` entry points or staged by torch).

Errors: ``ValueError`` (``InvalidArgument``) where the reference throws
std::invalid_argument, ``NumericFailure`` (with ``.iteration`` and ``.index``)
where it throws nlem::NumericFailure (types.hpp:20-31).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class NumericFailure(RuntimeError):
    """nlem::NumericFailure (proj/include/nlem/types.hpp:20-31)."""

    def __init__(self, message: str, iteration: int, index: int = -1):
        super().__init__(message)
        self.iteration = iteration
        self.index = index


class CudaError(RuntimeError):
    pass


def _raise(status: int, f: L.Failure):
    if status == L.NLEM_OK:
        return
    msg = f.message.decode(errors="replace")
    if status == L.NLEM_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == L.NLEM_NUMERIC_FAILURE:
        raise NumericFailure(msg, int(f.iteration), int(f.index))
    raise CudaError(msg or "CUDA error")


# ---- types (proj/include/nlem/types.hpp) --------------------------------------------
class BoxConstraint:
    """types.hpp:77-107."""

    def __init__(self, bounded=False, lower=-np.inf, upper=np.inf):
        self._bounded, self._lower, self._upper = bounded, lower, upper

    @staticmethod
    def unconstrained() -> "BoxConstraint":
        return BoxConstraint()

    @staticmethod
    def interval(lower: float, upper: float) -> "BoxConstraint":
        if not (lower <= upper):
            raise InvalidArgument("box requires lower <= upper")
        return BoxConstraint(True, float(lower), float(upper))

    def is_bounded(self):
        return self._bounded

    def lower(self):
        return self._lower

    def upper(self):
        return self._upper

    def c(self) -> L.Box:
        b = L.Box()
        b.bounded = 1 if self._bounded else 0
        b.lower = self._lower if self._bounded else 0.0
        b.upper = self._upper if self._bounded else 0.0
        return b


@dataclass
class AdmmConfig:
    """types.hpp:119-127."""

    mu: float = 1e-3
    max_iter: int = 100
    tol_primal: float = 0.0
    z_init: Optional[object] = None
    record_trace: bool = False


@dataclass
class IrlsConfig:
    """types.hpp:129-138."""

    epsilon: float = 1e-6
    max_iter: int = 100
    tol: float = 0.0
    x_init: Optional[object] = None
    record_trace: bool = False


@dataclass
class TraceRecord:
    iter: int
    objective: float
    primal_residual: float


@dataclass
class SolverResult:
    """types.hpp:143-149 (batched: arrays with a leading batch axis)."""

    minimizer: object
    objective: object
    iterations_run: object
    trace: list = field(default_factory=list)


DENOISE_SOLVERS = {"admm": L.SOLVER_ADMM, "irls": L.SOLVER_IRLS, "nlm_only": L.SOLVER_NLM_ONLY}
PATCH_INITS = {"noisy": L.INIT_NOISY_PATCH, "nlm": L.INIT_NLM_PATCH}


@dataclass
class NlemParams:
    """proj/include/nlem/nlem.hpp:23-35 (threads dropped; irls_tol = IrlsConfig::tol)."""

    search: int = 21
    patch: int = 7
    h: float = 0.0
    sigma: float = 0.0
    solver: str = "admm"
    solver_iters: int = 4
    mu: float = 1e-3
    epsilon: float = 1e-6
    init_mode: str = "noisy"
    range: BoxConstraint = field(default_factory=lambda: BoxConstraint.interval(0.0, 255.0))
    irls_tol: float = 0.0

    def c(self) -> L.ParamsC:
        p = L.ParamsC()
        p.search, p.patch, p.h, p.sigma = self.search, self.patch, self.h, self.sigma
        p.solver = DENOISE_SOLVERS[self.solver]
        p.solver_iters = self.solver_iters
        p.mu, p.epsilon = self.mu, self.epsilon
        p.init_mode = PATCH_INITS[self.init_mode]
        p.range = self.range.c()
        p.irls_tol = self.irls_tol
        return p


def default_init_mode(sigma: float) -> str:
    """proj/src/nlm.cpp:13-15."""
    return "noisy" if L.load().nlem_default_init_mode(sigma) == L.INIT_NOISY_PATCH else "nlm"


def validate(params: NlemParams) -> None:
    """proj/src/nlm.cpp:17-29."""
    f = L.Failure()
    _raise(L.load().nlem_validate_params(C.byref(params.c()), C.byref(f)), f)


# ---- device helpers --------------------------------------------------------------------
def _torch():
    import torch

    return torch


def _is_cuda(x) -> bool:
    try:
        torch = _torch()
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


def _dev(x, dtype=None, device=None):
    """Host/device array -> contiguous float32 CUDA tensor."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32)))
    t = t.to(device=device or ("cuda" if not t.is_cuda else t.device), dtype=dtype or torch.float32)
    return t.contiguous()


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(device):
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _out(host: bool, t):
    return t.cpu().numpy() if host else t


# ---- solvers ---------------------------------------------------------------------------
def admm_euclidean_median(points, weights, box: BoxConstraint | None = None,
                          cfg: AdmmConfig | None = None) -> SolverResult:
    """proj/include/nlem/admm.hpp:26-86 on a batch.

    points [B][n][d] (or one [n][d] problem), weights [B][n] (or [n]).
    """
    torch = _torch()
    box = box or BoxConstraint.unconstrained()
    cfg = cfg or AdmmConfig()
    host = not _is_cuda(points)
    P = _dev(points)
    single = P.dim() == 2
    if single:
        P = P.unsqueeze(0)
    if P.dim() != 3:
        raise InvalidArgument("points must be [n][d] or [batch][n][d]")
    B, n, d = P.shape
    dev = P.device
    Wt = _dev(weights, device=dev).reshape(B, -1)
    if Wt.shape[1] != n:
        raise InvalidArgument("weight count does not match point count")  # types.hpp:61-62
    zi = None
    if cfg.z_init is not None:
        zi = _dev(cfg.z_init, device=dev)
        if zi.shape[-1] != d:
            raise InvalidArgument("z_init dimension does not match point set")  # admm.hpp:32-34
        zi = zi.reshape(-1, d).expand(B, d).contiguous()
    z = torch.empty((B, d), device=dev, dtype=torch.float32)
    obj = torch.empty(B, device=dev, dtype=torch.float32)
    it = torch.empty(B, device=dev, dtype=torch.int32)
    T = int(cfg.max_iter)
    tro = trr = None
    if cfg.record_trace:
        tro = torch.full((B, T), float("nan"), device=dev)
        trr = torch.full((B, T), float("nan"), device=dev)
    c = L.AdmmConfigC()
    c.mu, c.max_iter, c.tol_primal = cfg.mu, T, cfg.tol_primal
    f = L.Failure()
    with torch.cuda.device(dev):
        st = L.load().nlem_admm_batched(_ptr(P), _ptr(Wt), B, n, d, _ptr(zi), box.c(), c, _ptr(z),
                                        _ptr(obj), _ptr(it), _ptr(tro), _ptr(trr), C.byref(f),
                                        _stream(dev))
    _raise(st, f)
    trace = []
    if cfg.record_trace:
        to, tr, its = tro.cpu().numpy(), trr.cpu().numpy(), it.cpu().numpy()
        trace = [[TraceRecord(t + 1, float(to[b, t]), float(tr[b, t])) for t in range(its[b])]
                 for b in range(B)]
    res = SolverResult(_out(host, z), _out(host, obj), _out(host, it), trace)
    if single:
        res.minimizer, res.objective, res.iterations_run = (
            res.minimizer[0], res.objective[0], res.iterations_run[0])
        res.trace = trace[0] if trace else []
    return res


def irls_euclidean_median(points, weights, cfg: IrlsConfig | None = None) -> SolverResult:
    """proj/include/nlem/irls.hpp:21-68 on a batch (unconstrained, like the reference)."""
    torch = _torch()
    cfg = cfg or IrlsConfig()
    host = not _is_cuda(points)
    P = _dev(points)
    single = P.dim() == 2
    if single:
        P = P.unsqueeze(0)
    B, n, d = P.shape
    dev = P.device
    Wt = _dev(weights, device=dev).reshape(B, -1)
    if Wt.shape[1] != n:
        raise InvalidArgument("weight count does not match point count")
    xi = None
    if cfg.x_init is not None:
        xi = _dev(cfg.x_init, device=dev)
        if xi.shape[-1] != d:
            raise InvalidArgument("x_init dimension does not match point set")
        xi = xi.reshape(-1, d).expand(B, d).contiguous()
    x = torch.empty((B, d), device=dev)
    obj = torch.empty(B, device=dev)
    it = torch.empty(B, device=dev, dtype=torch.int32)
    T = int(cfg.max_iter)
    tro = torch.full((B, T), float("nan"), device=dev) if cfg.record_trace else None
    c = L.IrlsConfigC()
    c.epsilon, c.max_iter, c.tol = cfg.epsilon, T, cfg.tol
    f = L.Failure()
    with torch.cuda.device(dev):
        st = L.load().nlem_irls_batched(_ptr(P), _ptr(Wt), B, n, d, _ptr(xi), c, _ptr(x), _ptr(obj),
                                        _ptr(it), _ptr(tro), C.byref(f), _stream(dev))
    _raise(st, f)
    trace = []
    if cfg.record_trace:
        to, its = tro.cpu().numpy(), it.cpu().numpy()
        trace = [[TraceRecord(t + 1, float(to[b, t]), float("nan")) for t in range(its[b])]
                 for b in range(B)]
    res = SolverResult(_out(host, x), _out(host, obj), _out(host, it), trace)
    if single:
        res.minimizer, res.objective, res.iterations_run = (
            res.minimizer[0], res.objective[0], res.iterations_run[0])
        res.trace = trace[0] if trace else []
    return res


# ---- images (proj/src/nlem.cpp, proj/src/nlm.cpp) -------------------------------------
def _image_call(noisy, params: NlemParams, frames: bool, entry: str):
    torch = _torch()
    host = not _is_cuda(noisy)
    X = _dev(noisy)
    if X.dim() != 2 or X.shape[0] < 1 or X.shape[1] < 1:
        raise InvalidArgument("image must be non-empty")
    H, W = X.shape
    dev = X.device
    out = torch.empty((H, W), device=dev)
    fr = torch.empty((params.solver_iters, H, W), device=dev) if frames else None
    f = L.Failure()
    pc = params.c()
    with torch.cuda.device(dev):
        if entry == "nlm":
            st = L.load().nlm_denoise(_ptr(X), H, W, C.byref(pc), _ptr(out), C.byref(f), _stream(dev))
        else:
            st = L.load().nlem_denoise(_ptr(X), H, W, C.byref(pc), _ptr(out), _ptr(fr), C.byref(f),
                                       _stream(dev))
    _raise(st, f)
    return _out(host, out), (_out(host, fr) if frames else None)


def nlem_denoise(noisy, params: NlemParams):
    """proj/include/nlem/nlem.hpp:71 (src/nlem.cpp:68-90)."""
    return _image_call(noisy, params, False, "nlem")[0]


def nlem_denoise_snapshots(noisy, params: NlemParams):
    """proj/include/nlem/nlem.hpp:76 (src/nlem.cpp:92-128): [solver_iters][H][W]."""
    return _image_call(noisy, params, True, "nlem")[1]


def nlm_denoise(noisy, params: NlemParams):
    """proj/include/nlem/nlem.hpp:65 (src/nlm.cpp:31-51)."""
    return _image_call(noisy, params, False, "nlm")[0]


def _host_out(out, shape):
    """A caller-supplied host output buffer must be a C-contiguous float32 array of `shape`
    (the C-ABI writes rows*cols floats through its pointer)."""
    if out is None:
        return np.empty(shape, np.float32)
    if not (isinstance(out, np.ndarray) and out.dtype == np.float32 and out.flags.c_contiguous
            and out.shape == tuple(shape) and out.flags.writeable):
        raise InvalidArgument(f"out must be a writeable C-contiguous float32 array of shape {tuple(shape)}")
    return out


def nlem_denoise_host(noisy: np.ndarray, params: NlemParams, out: np.ndarray | None = None,
                      device: int = 0) -> np.ndarray:
    """Host-buffer entry (nlem_denoise_host): H2D, kernels and D2H inside the call."""
    noisy = np.ascontiguousarray(noisy, dtype=np.float32)
    out = _host_out(out, noisy.shape)
    f = L.Failure()
    st = L.load().nlem_denoise_host(noisy.ctypes.data, noisy.shape[0], noisy.shape[1],
                                    C.byref(params.c()), out.ctypes.data, None, C.byref(f), device)
    _raise(st, f)
    return out


def nlem_denoise_multi_host(noisy: np.ndarray, params: NlemParams, devices, frames: bool = False):
    """Whole image over several devices (nlem_denoise_multi_host): one row band per entry of
    `devices` (entries may repeat), one host thread per band, no collective.  Returns out, or
    (out, frames [solver_iters][rows][cols]) with frames=True; bitwise equal to one device."""
    noisy = np.ascontiguousarray(noisy, dtype=np.float32)
    out = np.empty_like(noisy)
    fr = np.empty((params.solver_iters,) + noisy.shape, np.float32) if frames else None
    devs = (C.c_int32 * len(devices))(*[int(d) for d in devices])
    f = L.Failure()
    st = L.load().nlem_denoise_multi_host(noisy.ctypes.data, noisy.shape[0], noisy.shape[1],
                                          C.byref(params.c()), out.ctypes.data,
                                          fr.ctypes.data if frames else None, devs, len(devices),
                                          C.byref(f))
    _raise(st, f)
    return (out, fr) if frames else out


def nlem_denoise_rows_host(noisy_rows: np.ndarray, in_row0: int, rows: int, cols: int,
                           out_row0: int, out_rows: int, params: NlemParams,
                           out: np.ndarray | None = None, device: int = 0) -> np.ndarray:
    """Host-buffer row band (nlem_denoise_rows_host): H2D, kernels and D2H inside the call."""
    noisy_rows = np.ascontiguousarray(noisy_rows, dtype=np.float32)
    if noisy_rows.ndim != 2 or noisy_rows.shape[1] != cols:
        raise InvalidArgument("input rows must be [in_rows][cols]")
    out = _host_out(out, (out_rows, cols))
    f = L.Failure()
    st = L.load().nlem_denoise_rows_host(noisy_rows.ctypes.data, in_row0, noisy_rows.shape[0],
                                         rows, cols, out_row0, out_rows, C.byref(params.c()),
                                         out.ctypes.data, None, C.byref(f), device)
    _raise(st, f)
    return out


@dataclass
class PatchStack:
    """proj/include/nlem/patch.hpp:33-37 (patches [n][d] point-contiguous = Eigen d x n)."""

    patches: np.ndarray
    weights: np.ndarray
    self_column: int = -1


@dataclass
class PatchSolve:
    """proj/include/nlem/nlem.hpp:52-55."""

    init: np.ndarray
    patch: np.ndarray


def build_patch_stack(image: np.ndarray, row: int, col: int, search: int, k: int, h: float,
                      device: int = 0) -> PatchStack:
    """proj/src/patch.cpp:90-114 for one pixel of a host image (gathered on the GPU)."""
    image = np.ascontiguousarray(image, dtype=np.float32)
    if image.ndim != 2:
        raise InvalidArgument("image must be non-empty")
    pts = np.empty((search * search, k * k), np.float32)
    w = np.empty(search * search, np.float32)
    n, sc = C.c_int64(), C.c_int64()
    f = L.Failure()
    st = L.load().nlem_patch_stack_host(image.ctypes.data, image.shape[0], image.shape[1], row, col,
                                        search, k, h, pts.ctypes.data, w.ctypes.data, C.byref(n),
                                        C.byref(sc), C.byref(f), device)
    _raise(st, f)
    return PatchStack(pts[: n.value].copy(), w[: n.value].copy(), int(sc.value))


def solve_patch(stack: PatchStack, params: NlemParams, device: int = 0) -> PatchSolve:
    """proj/src/nlem.cpp:20-56 (init + ADMM / IRLS-then-clip / NlmOnly) on the GPU."""
    P = np.ascontiguousarray(stack.patches, dtype=np.float32)
    W = np.ascontiguousarray(stack.weights, dtype=np.float32)
    if P.ndim != 2 or W.shape != (P.shape[0],):
        raise InvalidArgument("weight count does not match point count")
    n, d = P.shape
    init = np.empty(d, np.float32)
    patch = np.empty(d, np.float32)
    f = L.Failure()
    st = L.load().nlem_solve_patch_host(P.ctypes.data, W.ctypes.data, n, d, stack.self_column,
                                        C.byref(params.c()), init.ctypes.data, patch.ctypes.data,
                                        C.byref(f), device)
    _raise(st, f)
    return PatchSolve(init, patch)


def band_halo(params: NlemParams) -> int:
    return int(L.load().nlem_band_halo(C.byref(params.c())))


def nlem_denoise_rows(noisy_rows, in_row0: int, rows: int, cols: int, out_row0: int,
                      out_rows: int, params: NlemParams, frames: bool = False):
    """One row band of a rows x cols image (global coordinates); device tensors in/out."""
    torch = _torch()
    X = _dev(noisy_rows)
    dev = X.device
    out = torch.empty((out_rows, cols), device=dev)
    fr = torch.empty((params.solver_iters, out_rows, cols), device=dev) if frames else None
    f = L.Failure()
    with torch.cuda.device(dev):
        st = L.load().nlem_denoise_rows(_ptr(X), in_row0, X.shape[0], rows, cols, out_row0,
                                        out_rows, C.byref(params.c()), _ptr(out), _ptr(fr),
                                        C.byref(f), _stream(dev))
    _raise(st, f)
    return (out, fr) if frames else out


# ---- SURVEY §8f "next" rows: device-side quality / certificate reductions -----------------
def frames_psnr(frames, clean) -> np.ndarray:
    """PSNR of every snapshot frame vs `clean` (psnr.hpp:12-24), reduced on the GPU in FP64."""
    torch = _torch()
    F = _dev(frames)
    Cl = _dev(clean, device=F.device)
    T = F.shape[0]
    count = Cl.numel()
    if F.numel() != T * count:
        raise InvalidArgument("frames and clean image sizes differ")
    out = np.empty(T, np.float64)
    f = L.Failure()
    with torch.cuda.device(F.device):
        st = L.load().nlem_frames_psnr(_ptr(F), _ptr(Cl), T, count, out.ctypes.data, C.byref(f),
                                       _stream(F.device))
    _raise(st, f)
    return out


def optimality_residual(points, weights, z, box: BoxConstraint | None = None):
    """Batched first-order certificate (diagnostics.hpp:22-55); 0 certifies optimality."""
    torch = _torch()
    box = box or BoxConstraint.unconstrained()
    host = not _is_cuda(points)
    P = _dev(points)
    if P.dim() == 2:
        P = P.unsqueeze(0)
    B, n, d = P.shape
    Wt = _dev(weights, device=P.device).reshape(B, n)
    Z = _dev(z, device=P.device).reshape(B, d)
    out = torch.empty(B, device=P.device)
    f = L.Failure()
    with torch.cuda.device(P.device):
        st = L.load().nlem_optimality_residual_batched(_ptr(P), _ptr(Wt), B, n, d, box.c(), _ptr(Z),
                                                       _ptr(out), C.byref(f), _stream(P.device))
    _raise(st, f)
    return _out(host, out)
