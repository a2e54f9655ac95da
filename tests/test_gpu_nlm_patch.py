"""GPU parity of the rows SURVEY §8 lists next to the solvers: nlm_denoise and the NlmOnly
solver (proj/src/nlm.cpp:31-51, proj/src/nlem.cpp:26-31) on noisy inputs, the single-pixel
drop-ins build_patch_stack / solve_patch (proj/src/patch.cpp:90-114, proj/src/nlem.cpp:20-56),
and smaller search windows (k=7 with S < 21, k=5 with S < 11: masked inside the low-rank / tile
kernels' grids by default, the exact p-form 'fast' image kernel when forced).  Every comparison is against the FP64 oracle on the same float32
input.  Bar: 1e-2 gray levels (north_star)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-2


@pytest.fixture(scope="module")
def nb():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1501_03879_b200 as nb

    return nb


def _psnr(a, clean):
    return 10 * math.log10(255 ** 2 / float(np.mean((a.astype(np.float64) - clean) ** 2)))


# ------------------------------------------------------------------ NLM and the NlmOnly solver
@pytest.mark.parametrize("cfg,k,S,sigma", [(0, 5, 11, 20.0), (2, 7, 21, 20.0)])
def test_nlm_denoise_vs_oracle(nb, oracle, cfg, k, S, sigma):
    """nlm_denoise (nlm.cpp:31-51: sum w a_centre / sum w, clipped) on the noisy config-0 and
    config-2 images, whole image; the reference's own check is a naive-loop NLM
    (test_denoise.cpp:41-72), restated by the oracle."""
    from paper_1501_03879_b200 import synth

    clean, noisy = synth.config_image(cfg)
    h = synth.reference_h(sigma, k * k)
    g = nb.NlemParams(search=S, patch=k, h=h, sigma=sigma, solver="admm", solver_iters=1)
    o = oracle.make_params(search=S, patch=k, h=h, sigma=sigma)
    gpu = nb.nlm_denoise(noisy, g)
    ref = oracle.nlm_denoise(noisy.astype(np.float64), o)
    assert np.abs(gpu - ref).max() <= TOL
    c = clean.astype(np.float64)
    assert abs(_psnr(gpu, c) - _psnr(ref, c)) <= 0.01


@pytest.mark.parametrize("cfg,k,S,sigma", [(0, 5, 11, 20.0), (2, 7, 21, 20.0)])
def test_nlm_only_solver_vs_oracle(nb, oracle, cfg, k, S, sigma):
    """DenoiseSolver::NlmOnly (nlem.cpp:26-31): the centre of the clipped weighted-mean patch
    (types.hpp:73 ratio form), whole noisy config-0 / config-2 images, both init modes (the
    init does not change the output), and its snapshots are the output repeated."""
    from paper_1501_03879_b200 import synth

    clean, noisy = synth.config_image(cfg)
    h = synth.reference_h(sigma, k * k)
    ref = None
    for init in ("noisy", "nlm"):
        g = nb.NlemParams(search=S, patch=k, h=h, sigma=sigma, solver="nlm_only", solver_iters=3,
                          init_mode=init)
        o = oracle.make_params(search=S, patch=k, h=h, sigma=sigma, solver="nlm", solver_iters=3,
                               init_mode=init)
        gpu = nb.nlem_denoise(noisy, g)
        if ref is None:
            ref = oracle.nlem_denoise(noisy.astype(np.float64), o)
        assert np.abs(gpu - ref).max() <= TOL
        frames = nb.nlem_denoise_snapshots(noisy, g)
        assert all((frames[t] == gpu).all() for t in range(3))
    c = clean.astype(np.float64)
    assert abs(_psnr(gpu, c) - _psnr(ref, c)) <= 0.01


# ------------------------------------------------------------------ single-pixel drop-ins
@pytest.mark.parametrize("row,col,S,k", [(0, 0, 7, 3), (5, 16, 7, 3), (9, 8, 21, 7), (19, 3, 21, 7),
                                         (2, 2, 11, 5)])
def test_build_patch_stack_vs_oracle(nb, oracle, row, col, S, k):
    """Clipped window, row-major neighbour order, self column, mirrored patches (bitwise: they
    are gathers of the same float32 samples) and weights (self weight exactly 1)."""
    rng = np.random.default_rng(row * 31 + col)
    img = (rng.uniform(0, 255, (20, 17))).astype(np.float32)
    h = 60.0 * k
    st = nb.build_patch_stack(img, row, col, S, k, h)
    P, w, sc = oracle.build_patch_stack(img.astype(np.float64), row, col, S, k, h)
    assert st.self_column == sc and st.patches.shape == P.shape
    assert (st.patches.astype(np.float64) == P).all()
    assert st.weights[st.self_column] == 1.0
    np.testing.assert_allclose(st.weights, w, rtol=2e-5)


def test_build_patch_stack_errors(nb):
    img = np.zeros((6, 5), np.float32)
    with pytest.raises(nb.InvalidArgument, match="pixel outside the image"):
        nb.build_patch_stack(img, 6, 0, 7, 3, 10.0)
    with pytest.raises(nb.InvalidArgument, match="search window must be odd and positive"):
        nb.build_patch_stack(img, 0, 0, 6, 3, 10.0)
    with pytest.raises(nb.InvalidArgument, match="patch size must be odd and positive"):
        nb.build_patch_stack(img, 0, 0, 7, 0, 10.0)
    with pytest.raises(nb.InvalidArgument, match="bandwidth h must be positive"):
        nb.build_patch_stack(img, 0, 0, 7, 3, 0.0)
    bad = img.copy()
    bad[1, 1] = np.nan
    with pytest.raises(nb.InvalidArgument, match="intensities must be finite"):
        nb.build_patch_stack(bad, 0, 0, 7, 3, 10.0)


@pytest.mark.parametrize("solver", ["admm", "irls", "nlm_only"])
@pytest.mark.parametrize("init", ["noisy", "nlm"])
def test_solve_patch_vs_oracle(nb, oracle, solver, init):
    """solve_patch (nlem.cpp:20-56) on config-3-parameter stacks (k=7, S=21) of a noisy crop:
    init = the self column or the weighted mean; ADMM from the init (tol 0), IRLS from the init
    (tol < 0: fixed count) then clipped, NlmOnly = the clipped weighted mean.  The centre
    coordinate of `patch` is what nlem_denoise writes (nlem.cpp:84)."""
    from paper_1501_03879_b200 import synth

    _, noisy = synth.noisy_image(40, 40, 8, 5, 30.0)
    h = synth.reference_h(30.0, 49)
    p = nb.NlemParams(search=21, patch=7, h=h, solver=solver, solver_iters=10, mu=1.0,
                      epsilon=1e-4, init_mode=init, irls_tol=-1.0)
    full = nb.nlem_denoise(noisy, p)
    for r, c in ((0, 0), (20, 17), (39, 30)):
        st = nb.build_patch_stack(noisy, r, c, 21, 7, h)
        res = nb.solve_patch(st, p)
        P = st.patches.astype(np.float64)
        w = st.weights.astype(np.float64)
        init_ref = oracle.initial_patch(P, w, st.self_column, 0 if init == "noisy" else 1)
        np.testing.assert_allclose(res.init, init_ref, atol=1e-3)
        if solver == "nlm_only":
            ref = np.clip(oracle.initial_patch(P, w, st.self_column, 1), 0.0, 255.0)
        elif solver == "admm":
            ref = oracle.admm_batched(P[None], w[None], mu=1.0, max_iter=10, z_init=init_ref,
                                      box=(0.0, 255.0)).minimizer[0]
        else:
            ref = np.clip(oracle.irls_batched(P[None], w[None], epsilon=1e-4, max_iter=10, tol=-1.0,
                                              x_init=init_ref).minimizer[0], 0.0, 255.0)
        assert np.abs(res.patch - ref).max() <= TOL, (solver, init, r, c)
        assert res.patch.min() >= 0.0 and res.patch.max() <= 255.0
        # the image kernels write the centre coordinate of the same solve
        assert abs(float(res.patch[24]) - float(full[r, c])) <= TOL


def test_solve_patch_errors(nb):
    st = nb.PatchStack(np.zeros((3, 4), np.float32), np.ones(3, np.float32), 3)
    p = nb.NlemParams(search=3, patch=3, h=10.0, solver_iters=2)
    with pytest.raises(nb.InvalidArgument, match="no valid self column"):
        nb.solve_patch(st, p)
    st.self_column = 0
    with pytest.raises(nb.InvalidArgument, match="penalty mu must be positive"):
        nb.solve_patch(st, nb.NlemParams(search=3, patch=3, h=10.0, mu=0.0))
    st.weights = -st.weights
    with pytest.raises(nb.InvalidArgument, match="finite and nonnegative"):
        nb.solve_patch(st, p)


# ------------------------------------------------- smaller search windows (k = 7 / k = 5)
@pytest.mark.parametrize("k,S", [(7, 15), (7, 19), (5, 9), (5, 7)])
@pytest.mark.parametrize("shape", [(33, 29), (6, 40)])
@pytest.mark.parametrize("force", ["", "fast"])
def test_small_window_shapes_vs_oracle(nb, oracle, monkeypatch, k, S, shape, force):
    """k = 7 with S < 21 and k = 5 with S < 11.  Default dispatch: the low-rank / tile kernels run
    the smaller window MASKED inside their fixed 21 x 21 / 11 x 11 grid (zero-weight points
    outside it, a padded-band border of the grid's size).  NLEM_KERNEL=fast: nlem_pixels_fast
    (exact p-form, patch stack in shared memory), the previous route for these shapes.  Ragged
    images (rows < S) included.  ADMM and NlmOnly, every frame vs the oracle."""
    if force:
        monkeypatch.setenv("NLEM_KERNEL", force)  # read per call
    rng = np.random.default_rng(k * 100 + S)
    img = (rng.uniform(0, 255, shape) + rng.normal(0, 25, shape)).astype(np.float32)
    h = 25.0 * 10 * k
    for solver in ("admm", "nlm_only"):
        g = nb.NlemParams(search=S, patch=k, h=h, solver=solver, solver_iters=6, mu=1.0,
                          init_mode="nlm")
        o = oracle.make_params(search=S, patch=k, h=h, solver={"nlm_only": "nlm"}.get(solver, solver),
                               solver_iters=6, mu=1.0, init_mode="nlm")
        fg = nb.nlem_denoise_snapshots(img, g)
        _, fo = oracle.nlem_denoise(img.astype(np.float64), o, snapshots=True)
        assert np.abs(fg - fo).max() <= TOL, (solver, k, S, shape, force)


@pytest.mark.parametrize("k,S", [(7, 7), (7, 11), (7, 13), (7, 17), (5, 5), (5, 13), (5, 21),
                                 (3, 3), (3, 9), (3, 11), (3, 15), (3, 21)])
def test_masked_window_all_solvers_and_bands(nb, oracle, k, S):
    """Every odd patch side up to 7 with windows up to 21 is served by the low-rank kernel (k = 7) or
    a tile-kernel instantiation (k = 7 / 5 / 3 on a 21 x 21 or 11 x 11 grid), smaller windows masked.
    Masked windows through every solver of the low-rank / tile kernels (ADMM at mu = 1, ADMM at
    mu = 1e-3 with 8 sweeps - the hand-off to the exact tile kernel -, IRLS, NlmOnly; noisy and
    NLM init) vs the oracle, and a 3-band split with S/2 + k/2 halo rows (less than the kernels'
    fixed tile border: the band padding clamps) bitwise equal to the whole-image call."""
    import torch

    rng = np.random.default_rng(1000 + 31 * k + S)
    img = (rng.uniform(0, 255, (40, 37)) + rng.normal(0, 20, (40, 37))).astype(np.float32)
    h = 20.0 * 10 * k
    cases = [dict(solver="admm", mu=1.0, init_mode="nlm", solver_iters=6),
             dict(solver="admm", mu=1e-3, init_mode="noisy", solver_iters=8),
             dict(solver="irls", epsilon=1e-4, irls_tol=-1.0, init_mode="nlm", solver_iters=6),
             dict(solver="nlm_only", init_mode="nlm", solver_iters=3)]
    for kw in cases:
        g = nb.NlemParams(search=S, patch=k, h=h, **kw)
        okw = dict(kw, solver={"nlm_only": "nlm"}.get(kw["solver"], kw["solver"]))
        o = oracle.make_params(search=S, patch=k, h=h, **okw)
        fg = nb.nlem_denoise_snapshots(img, g)
        _, fo = oracle.nlem_denoise(img.astype(np.float64), o, snapshots=True)
        assert np.abs(fg - fo).max() <= TOL, (kw, k, S)
    g = nb.NlemParams(search=S, patch=k, h=h, **cases[0])
    X = torch.from_numpy(img).cuda()
    whole = nb.nlem_denoise(X, g).cpu().numpy()
    halo = S // 2 + k // 2
    parts = []
    for r0, r1 in ((0, 13), (13, 27), (27, 40)):
        a0, a1 = max(0, r0 - halo), min(40, r1 + halo)
        parts.append(nb.nlem_denoise_rows(X[a0:a1].contiguous(), a0, 40, 37, r0, r1 - r0, g).cpu().numpy())
    assert np.array_equal(np.concatenate(parts), whole)
