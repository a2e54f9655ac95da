"""Pins the FP64 CPU oracle (oracle/nlem_oracle.cpp) against every known-answer
test and property test the reference's own unit tests hold for the path
(tests/golden/reference_kats.json + the procedural checks of
proj/tests/unit/test_{patch,prox,costs,solvers,denoise,noise}.cpp).
CPU only."""
import math

import numpy as np
import pytest

from tests.support import fold_index, house_like, kats, random_instance

K = kats()


def test_mirror_index_kats(oracle):
    for i, n, e in K["mirror_index"]["cases"]:
        assert oracle.mirror_index(i, n) == e


def test_mirror_index_matches_fold(oracle):  # test_patch.cpp:33-42
    for n in (1, 2, 3, 5, 8):
        for i in range(-25, 26):
            assert oracle.mirror_index(i, n) == fold_index(i, n)


def test_corner_patch_kat(oracle):
    k = K["corner_patch_2x2"]
    p = oracle.patch_at(np.array(k["image"], float), k["row"], k["col"], k["k"])
    assert p.tolist() == k["expected"]


def test_interior_patch_verbatim(oracle):  # test_patch.cpp:61-73
    img = np.fromfunction(lambda r, c: 3.0 * r + 7.0 * c, (9, 11))
    p = oracle.patch_at(img, 4, 5, 3)
    exp = [3.0 * (4 + dr) + 7.0 * (5 + dc) for dr in (-1, 0, 1) for dc in (-1, 0, 1)]
    assert p.tolist() == exp


def test_patch_side_validated(oracle):  # test_patch.cpp:81-86
    img = np.zeros((4, 4))
    for k in (4, -3, 0):
        with pytest.raises(oracle.OracleError):
            oracle.patch_at(img, 0, 0, k)


def test_weights_kats(oracle):
    k = K["weights_exp_minus_one"]
    w = oracle.patch_weights(np.array(k["patches"], float), k["center"], k["h"])
    assert w[0] == 1.0
    assert w[1] == pytest.approx(k["expected"][1], rel=k["rel_tol"])
    with pytest.raises(oracle.OracleError):
        oracle.patch_weights(np.zeros((3, 4)), 0, 0.0)


def test_weights_long_double_recompute(oracle):  # test_patch.cpp:127-141
    rng = np.random.default_rng(83)
    img = rng.uniform(0, 255, size=(5, 8))
    pats = np.stack([oracle.patch_at(img, r, c, 3) for r in range(5) for c in range(8)])
    w = oracle.patch_weights(pats, 21, 37.5)
    sq = ((pats.astype(np.longdouble) - pats[21].astype(np.longdouble)) ** 2).sum(axis=1)
    exp = np.exp(-sq / (np.longdouble(37.5) ** 2)).astype(np.float64)
    np.testing.assert_allclose(w, exp, rtol=1e-12)
    assert w[21] == 1.0


def test_corner_and_interior_stack(oracle):
    k = K["corner_stack"]
    rng = np.random.default_rng(84)
    img = rng.uniform(0, 255, size=(k["rows"], k["cols"]))
    pats, w, sc = oracle.build_patch_stack(img, k["row"], k["col"], k["search"], k["k"], 20.0)
    assert pats.shape[0] == k["expected_n"] and sc == k["expected_self_column"] and w[0] == 1.0
    for i, (r, c) in enumerate(k["expected_neighbours"]):
        assert pats[i].tolist() == oracle.patch_at(img, r, c, 3).tolist()
    k = K["interior_stack"]
    img = rng.uniform(0, 255, size=(k["rows"], k["cols"]))
    pats, w, sc = oracle.build_patch_stack(img, k["row"], k["col"], k["search"], k["k"], 20.0)
    assert pats.shape[0] == k["expected_n"] and sc == k["expected_self_column"] and w[sc] == 1.0


def test_prox_kats(oracle):
    k = K["prox_far_unit_pull"]
    x = oracle.prox_weighted_norm(k["v"], k["u"], k["lambda"])
    np.testing.assert_allclose(x, k["expected"], rtol=1e-15)
    k = K["prox_lands_on_u"]
    for lam in k["lambdas"]:
        lam = math.inf if lam == "inf" else lam
        assert oracle.prox_weighted_norm(k["v"], k["u"], lam).tolist() == k["expected"]
    k = K["prox_zero_pull_identity"]
    assert oracle.prox_weighted_norm(k["v"], k["u"], 0.0).tolist() == k["expected"]
    k = K["prox_v_equals_u"]
    assert oracle.prox_weighted_norm(k["v"], k["u"], k["lambda"]).tolist() == k["expected"]
    for bad in (-1e-12, float("nan")):
        with pytest.raises(oracle.OracleError):
            oracle.prox_weighted_norm([3.0, 4.0], [0.0, 0.0], bad)


def test_prox_segment_and_moreau(oracle):  # test_prox.cpp:56-94
    rng = np.random.default_rng(12)
    for trial in range(500):
        d = 1 + trial % 16
        v = 3 * rng.standard_normal(d)
        u = 3 * rng.standard_normal(d)
        lam = abs(rng.standard_normal())
        if trial % 5 == 0:
            lam = 0.0
        if trial % 7 == 0:
            lam = 2.0 * np.linalg.norm(v - u)
        s = oracle.prox_weighted_norm(v, u, lam) + oracle.project_ball(v - u, lam)
        assert np.linalg.norm(s - v) <= 1e-12 * (1 + np.linalg.norm(v))
        dist = np.linalg.norm(v - u)
        t = 0.0 if dist == 0 else min(lam, dist) / dist
        x = oracle.prox_weighted_norm(v, u, lam)
        assert np.linalg.norm(x - (v + t * (u - v))) <= 1e-12 * (1 + np.linalg.norm(v) + np.linalg.norm(u))


def test_ball_and_box(oracle):
    for c in K["ball_projection"]["cases"]:
        np.testing.assert_allclose(oracle.project_ball(c["y"], c["radius"]), c["expected"], rtol=1e-15)


def test_costs_kats(oracle):
    k = K["em_cost_345"]
    assert oracle.em_cost(k["points"], k["weights"], k["x"]) == pytest.approx(5.0, rel=1e-15)
    k = K["surrogate_at_point"]
    assert oracle.surrogate_cost(k["points"], k["weights"], k["x"], k["eps"]) == 1.0


def test_em_cost_long_double(oracle):  # test_costs.cpp:44-61
    rng = np.random.default_rng(21)
    x = np.array([0.3, 0.8, -0.2])
    for _ in range(50):
        pts = rng.uniform(0, 1, size=(5, 3))
        w = rng.uniform(0.1, 2.0, size=5)
        exp = (w.astype(np.longdouble) * np.sqrt(((x.astype(np.longdouble) - pts) ** 2).sum(1))).sum()
        assert oracle.em_cost(pts, w, x) == pytest.approx(float(exp), rel=1e-12)


def _admm1(oracle, k, **kw):
    pts = np.array(k["points"], float)[None]
    w = np.array(k["weights"], float)[None]
    zi = None if k.get("z_init") is None else np.array(k["z_init"], float)[None]
    return oracle.admm_batched(pts, w, mu=k["mu"], max_iter=k["max_iter"],
                               tol_primal=k.get("tol_primal", 0.0), z_init=zi, **kw)


def test_admm_single_point_kats(oracle):
    k = K["admm_single_point_distant_start"]
    r = _admm1(oracle, k)
    assert r.iterations[0] == 1 and np.linalg.norm(r.minimizer[0]) == 0.0 and r.objective[0] == 0.0
    k = K["admm_single_point_undersized_radius"]
    r = _admm1(oracle, k)
    assert r.iterations[0] == 1 and r.objective[0] == pytest.approx(3.0, rel=1e-12)
    k = K["admm_single_point_default_start"]
    r = _admm1(oracle, k)
    assert r.minimizer[0].tolist() == k["expected_minimizer"] and r.objective[0] == 0.0


def test_admm_triangle(oracle):
    k = K["admm_equilateral_triangle"]
    r = _admm1(oracle, k)
    np.testing.assert_allclose(r.minimizer[0], k["expected_minimizer"], rtol=k["rel_tol"])
    assert r.objective[0] == pytest.approx(k["expected_objective"], rel=k["objective_rel_tol"])


def test_admm_recursion_kat(oracle):
    k = K["admm_recursion"]
    r = _admm1(oracle, k, trace=True)
    assert r.trace_objective[0, :2].tolist() == k["expected_trace_objective"]
    assert r.trace_residual[0, :2].tolist() == k["expected_trace_residual"]
    assert r.trace_residual[0, 2] <= k["third_residual_max"]
    assert r.minimizer[0, 0] == pytest.approx(0.5, rel=1e-12)
    assert r.objective[0] == pytest.approx(1.0, rel=1e-12)


def test_admm_1d_exhaustive(oracle):  # test_solvers.cpp:287-302
    rng = np.random.default_rng(37)
    for _ in range(10):
        n = 3 + int(rng.integers(0, 20))
        pts, w = random_instance(rng, n, 1)
        best = min(oracle.em_cost(pts, w, pts[k]) for k in range(n))
        r = oracle.admm_batched(pts[None], w[None], mu=2 * w.mean(), max_iter=100000)
        assert abs(r.objective[0] - best) <= 1e-9


def test_admm_box_holds_and_residual_falls(oracle):  # test_solvers.cpp:254-273
    rng = np.random.default_rng(35)
    for _ in range(10):
        n = 5 + int(rng.integers(0, 20))
        d = 2 + int(rng.integers(0, 4))
        pts, w = random_instance(rng, n, d)
        r = oracle.admm_batched(pts[None], w[None], mu=2 * w.mean(), max_iter=50, box=(0.2, 0.8),
                                trace=True)
        assert r.trace_residual[0, -1] < r.trace_residual[0, 0]
        z = r.minimizer[0]
        assert (z >= 0.2).all() and (z <= 0.8).all()


def test_irls_kats(oracle):
    k = K["irls_single_point"]
    r = oracle.irls_batched(np.array(k["points"])[None], np.array(k["weights"])[None],
                            epsilon=k["epsilon"], max_iter=k["max_iter"])
    assert np.linalg.norm(r.minimizer[0] - 2.5) <= 1e-15 * np.linalg.norm([2.5] * 3)
    assert r.iterations[0] == 1
    k = K["irls_equilateral_corner_start"]
    r = oracle.irls_batched(np.array(k["points"])[None], np.array(k["weights"], float)[None],
                            epsilon=k["epsilon"], max_iter=k["max_iter"],
                            x_init=np.array(k["x_init"])[None])
    np.testing.assert_allclose(r.minimizer[0], k["expected_minimizer"], rtol=k["rel_tol"])


def test_irls_surrogate_non_increasing(oracle):  # test_solvers.cpp:194-212
    rng = np.random.default_rng(32)
    for _ in range(20):
        n = 4 + int(rng.integers(0, 30))
        d = 1 + int(rng.integers(0, 5))
        pts, w = random_instance(rng, n, d)
        r = oracle.irls_batched(pts[None], w[None], epsilon=1e-6, max_iter=100,
                                x_init=np.zeros((1, d)), trace=True)
        t = r.trace_objective[0, : r.iterations[0]]
        assert (t[1:] <= t[:-1] * (1 + 1e-12)).all()


def test_irls_matches_admm(oracle):  # test_solvers.cpp:214-223
    rng = np.random.default_rng(33)
    pts, w = random_instance(rng, 12, 2)
    a = oracle.irls_batched(pts[None], w[None], epsilon=1e-6, max_iter=200)
    b = oracle.admm_batched(pts[None], w[None], mu=2 * w.mean(), max_iter=100000)
    assert abs(a.objective[0] - b.objective[0]) <= 1e-6 * b.objective[0]


def test_overflow_raises_numeric_failure(oracle):  # test_solvers.cpp:342-368
    k = K["admm_overflow"]
    with pytest.raises(oracle.OracleError) as e:
        _admm1(oracle, k, trace=True)
    assert e.value.status == 2 and e.value.iteration >= 1 and "objective" in str(e.value)
    with pytest.raises(oracle.OracleError) as e:
        oracle.irls_batched(np.array(k["points"])[None], np.array(k["weights"])[None],
                            epsilon=1e-6, max_iter=5)
    assert e.value.status == 2


def test_solver_validation(oracle):  # test_solvers.cpp:370-395
    pts = np.zeros((1, 1, 2))
    w = np.ones((1, 1))
    with pytest.raises(oracle.OracleError) as e:
        oracle.admm_batched(pts, w, mu=0.0, max_iter=10)
    assert e.value.status == 1
    with pytest.raises(oracle.OracleError):
        oracle.irls_batched(pts, w, epsilon=0.0, max_iter=10)
    with pytest.raises(oracle.OracleError):
        oracle.admm_batched(np.zeros((1, 0, 2)), np.zeros((1, 0)), mu=1.0, max_iter=10)


def _small(oracle, solver, **kw):  # test_denoise.cpp:74-84
    base = dict(search=7, patch=3, h=30.0, sigma=15.0, solver=solver, solver_iters=4, threads=1)
    base.update(kw)
    return oracle.make_params(**base)


def test_constant_image_fixed_point(oracle):
    k = K["nlem_constant_image"]
    img = np.full((k["rows"], k["cols"]), k["value"])
    assert (oracle.nlem_denoise(img, _small(oracle, "admm")) == 77.0).all()
    assert (oracle.nlm_denoise(img, _small(oracle, "admm")) == 77.0).all()
    assert np.abs(oracle.nlem_denoise(img, _small(oracle, "irls")) - 77.0).max() <= 1e-9
    assert np.abs(oracle.nlem_denoise(img, _small(oracle, "nlm")) - 77.0).max() <= 1e-9


def test_vanishing_bandwidth_identity(oracle):  # test_denoise.cpp:195-212
    img = np.round(house_like(12))
    assert (oracle.nlm_denoise(img, _small(oracle, "admm", h=1e-6)) == img).all()
    assert np.abs(oracle.nlem_denoise(img, _small(oracle, "admm", h=1e-6)) - img).max() <= 1e-9
    assert np.abs(oracle.nlem_denoise(img, _small(oracle, "irls", h=1e-6)) - img).max() <= 1e-9


def test_box_prior_respected(oracle):  # test_denoise.cpp:214-226
    noisy = oracle.add_gaussian_noise(house_like(12), 25.0, 9)
    for s in ("admm", "irls", "nlm"):
        out = oracle.nlem_denoise(noisy, _small(oracle, s, box=(100.0, 140.0)))
        assert out.min() >= 100.0 and out.max() <= 140.0


def test_snapshots_equal_truncated_runs(oracle):  # test_denoise.cpp:264-280
    noisy = oracle.add_gaussian_noise(house_like(10), 20.0, 11)
    for s in ("admm", "irls"):
        p = _small(oracle, s, solver_iters=3)
        _, frames = oracle.nlem_denoise(noisy, p, snapshots=True)
        for t in (1, 2, 3):
            direct = oracle.nlem_denoise(noisy, _small(oracle, s, solver_iters=t))
            assert (frames[t - 1] == direct).all()


def test_snapshots_forward_fill(oracle):  # test_denoise.cpp:282-290
    img = np.full((8, 8), 50.0)
    _, frames = oracle.nlem_denoise(img, _small(oracle, "admm", solver_iters=4), snapshots=True)
    assert (frames == 50.0).all()


def test_thread_count_invariance(oracle):  # test_denoise.cpp:242-262
    noisy = oracle.add_gaussian_noise(house_like(14), 20.0, 3)
    for s in ("admm", "irls", "nlm"):
        a = oracle.nlem_denoise(noisy, _small(oracle, s, threads=1))
        b = oracle.nlem_denoise(noisy, _small(oracle, s, threads=4))
        assert (a == b).all()


def test_patchwise_mean_equals_nlm(oracle):  # test_denoise.cpp:228-240
    noisy = oracle.add_gaussian_noise(house_like(12), 18.0, 6)
    p = _small(oracle, "nlm")
    np.testing.assert_allclose(oracle.nlem_denoise(noisy, p), oracle.nlm_denoise(noisy, p), rtol=1e-12)


def test_failure_carries_pixel(oracle):  # test_denoise.cpp:323-338
    img = np.fromfunction(lambda r, c: np.where((r + c) % 2 == 0, 0.0, 1e200), (8, 8))
    with pytest.raises(oracle.OracleError) as e:
        oracle.nlem_denoise(img, _small(oracle, "irls", box=None))
    assert "pixel (" in str(e.value) and e.value.status == 2


def test_noise_kats(oracle):  # test_noise.cpp
    clean = house_like(32)
    assert (oracle.add_gaussian_noise(clean, 0.0, 12345) == clean).all()
    a = oracle.add_gaussian_noise(clean, 15.0, 7)
    assert (a == oracle.add_gaussian_noise(clean, 15.0, 7)).all()
    assert (a != oracle.add_gaussian_noise(clean, 15.0, 8)).any()
    bright = oracle.add_gaussian_noise(np.full((48, 48), 250.0), 30.0, 4)
    assert bright.max() > 255.0  # not clipped
    k = K["noise_psnr_closed_form"]
    clean = house_like(128)
    noisy = oracle.add_gaussian_noise(clean, k["sigma"], k["seed"])
    assert oracle.psnr(clean, noisy) == pytest.approx(k["expected_psnr"], rel=0.01)
