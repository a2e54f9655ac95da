"""Edge cases of the generic (any n, d) kernels: point sets and search windows whose work
block (2n prox scales and weights) exceeds shared memory run from a global-memory slab
(the reference accepts any n, proj/include/nlem/types.hpp:58-68)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nb():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1501_03879_b200 as nb

    return nb


@pytest.mark.parametrize("n,d", [(50000, 2), (40000, 20)])
def test_huge_point_sets_vs_oracle(nb, oracle, n, d):
    rng = np.random.default_rng(n + d)
    pts = rng.uniform(0, 1, size=(2, n, d)).astype(np.float32)
    w = rng.uniform(0.5, 1.5, size=(2, n)).astype(np.float32)
    r = nb.admm_euclidean_median(pts, w, nb.BoxConstraint.interval(0.2, 0.9),
                                 nb.AdmmConfig(mu=2.0, max_iter=15, tol_primal=-1.0))
    ref = oracle.admm_batched(pts.astype(np.float64), w.astype(np.float64), mu=2.0, max_iter=15,
                              tol_primal=-1.0, box=(0.2, 0.9))
    assert np.abs(r.minimizer - ref.minimizer).max() <= 1e-4
    np.testing.assert_allclose(r.objective, ref.objective, rtol=1e-4)
    ir = nb.irls_euclidean_median(pts, w, nb.IrlsConfig(epsilon=1e-4, max_iter=10, tol=-1.0))
    iref = oracle.irls_batched(pts.astype(np.float64), w.astype(np.float64), epsilon=1e-4,
                               max_iter=10, tol=-1.0)
    assert np.abs(ir.minimizer - iref.minimizer).max() <= 1e-4


def test_huge_search_window_vs_oracle(nb, oracle):
    """S = 301 (S^2 = 90,601 window slots): the generic NLEM kernel's stack, state and work all
    live in the global slab; on a 10 x 12 image the clipped window is the whole image."""
    rng = np.random.default_rng(7)
    img = (rng.uniform(0, 255, (10, 12))).astype(np.float32)
    g = nb.NlemParams(search=301, patch=3, h=300.0, solver="admm", solver_iters=5, mu=1.0,
                      init_mode="nlm")
    o = oracle.make_params(search=301, patch=3, h=300.0, solver="admm", solver_iters=5, mu=1.0,
                           init_mode="nlm")
    out = nb.nlem_denoise(img, g)
    ref = oracle.nlem_denoise(img.astype(np.float64), o)
    assert np.abs(out - ref).max() <= 1e-2
