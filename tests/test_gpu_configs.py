"""GPU parity at the BASELINE.json configurations as specified (not crops): the benchmarked
config 3 (4096^2, sigma 30, k=7, S=21, T=10) on full-width rows at both image edges and in
the interior, and config 4 (512^2, sigma 10/20/40/60, ADMM and IRLS T=1..100) on
stride-sampled rows with PSNR per iteration.  The oracle is the FP64 restatement of
proj/src/nlem.cpp:68-128 on the same float32 inputs.  Bar (north_star): max |GPU - oracle|
<= 1e-2 gray levels and |dPSNR| <= 0.01 dB."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-2
PSNR_TOL = 0.01


def _psnr(a, clean):
    return 10 * math.log10(255 ** 2 / float(np.mean((a.astype(np.float64) - clean) ** 2)))


@pytest.fixture(scope="module")
def nb():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1501_03879_b200 as nb

    return nb


@pytest.fixture(scope="module")
def config3(nb):
    """The whole benchmarked image through the production dispatch (low-rank kernel + exact
    hand-off), once for the module."""
    import torch

    from paper_1501_03879_b200 import synth

    clean, noisy = synth.config_image(3)
    p = nb.NlemParams(search=21, patch=7, h=synth.reference_h(30.0, 49), sigma=30.0, solver="admm",
                      solver_iters=10, mu=1.0, init_mode="nlm")
    out = nb.nlem_denoise(torch.from_numpy(noisy).cuda(), p).cpu().numpy()
    return clean, noisy, out


def test_config3_rows_vs_oracle(nb, oracle, config3):
    """Rows 0-3 (clipped windows, mirrored patches at the top), three interior rows and rows
    4092-4095 (bottom), full width (4096 pixels each, both side edges included)."""
    from paper_1501_03879_b200 import synth

    clean, noisy, out = config3
    o = oracle.make_params(search=21, patch=7, h=synth.reference_h(30.0, 49), sigma=30.0,
                           solver="admm", solver_iters=10, mu=1.0, init_mode="nlm")
    X = noisy.astype(np.float64)
    rows = [0, 1, 2, 3, 1337, 2048, 3071, 4092, 4093, 4094, 4095]
    ref = {}
    for r0, r1 in ((0, 4), (1337, 1338), (2048, 2049), (3071, 3072), (4092, 4096)):
        full = oracle.nlem_denoise(X, o, rows=(r0, r1))
        for r in range(r0, r1):
            ref[r] = full[r]
    g = out[rows].astype(np.float64)
    f = np.stack([ref[r] for r in rows])
    err = np.abs(g - f)
    assert err.max() <= TOL, (err.max(), np.unravel_index(err.argmax(), err.shape))
    c = clean[rows].astype(np.float64)
    assert abs(_psnr(g, c) - _psnr(f, c)) <= PSNR_TOL


def test_config3_reference_default_mu_rows_vs_oracle(nb, oracle):
    """The benchmarked image at the reference's default penalty mu = 1e-3 (types.hpp:121), T = 10:
    the small-mu probe routes the band to the exact p-form tile kernel.  A top band (clipped
    windows), an interior band and a bottom band of the 4096-wide image, full width, against the
    oracle on the same rows."""
    import torch

    from paper_1501_03879_b200 import synth

    clean, noisy = synth.config_image(3)
    kw = dict(search=21, patch=7, h=synth.reference_h(30.0, 49), sigma=30.0, solver="admm",
              solver_iters=10, mu=1e-3, init_mode="nlm")
    p = nb.NlemParams(**kw)
    o = oracle.make_params(**kw)
    X = torch.from_numpy(noisy).cuda()
    Xd = noisy.astype(np.float64)
    worst = 0.0
    for r0, r1 in ((0, 2), (2047, 2049), (4094, 4096)):
        a0, a1 = max(0, r0 - 13), min(4096, r1 + 13)  # band + halo, global coordinates
        g = nb.nlem_denoise_rows(X[a0:a1].contiguous(), a0, 4096, 4096, r0, r1 - r0, p).cpu().numpy()
        f = oracle.nlem_denoise(Xd, o, rows=(r0, r1))[r0:r1]
        worst = max(worst, float(np.abs(g.astype(np.float64) - f).max()))
    assert worst <= TOL, worst


def test_config3_whole_image_sanity(config3):
    """Every pixel finite and inside the box; denoising raises PSNR over the noisy input."""
    clean, noisy, out = config3
    assert np.isfinite(out).all() and out.min() >= 0.0 and out.max() <= 255.0
    c = clean.astype(np.float64)
    assert _psnr(out, c) > _psnr(noisy, c) + 5.0


@pytest.mark.parametrize("sigma", [10.0, 20.0, 40.0, 60.0])
def test_config4_sweep_vs_oracle(nb, oracle, sigma):
    """Config 4: 512^2 (config-2 generator) at sigma, ADMM (mu=1, NLM init) and IRLS (eps=1e-4,
    tol<0: a fixed count) emitting all 100 frames in one run as
    nlem_denoise_snapshots does; every frame of 10 sampled rows (0, 511 and stride 57) matches
    the oracle and the PSNR of the sample against the clean image agrees per iteration."""
    from paper_1501_03879_b200 import synth

    clean, noisy = synth.config_image(2, sigma=sigma)
    h = synth.reference_h(sigma, 49)
    rows = sorted({0, 511} | set(range(29, 512, 57)))
    X = noisy.astype(np.float64)
    c = clean[rows].astype(np.float64)
    for solver, kw in (("admm", dict(mu=1.0)), ("irls", dict(epsilon=1e-4, irls_tol=-1.0))):
        g = nb.NlemParams(search=21, patch=7, h=h, sigma=sigma, solver=solver, solver_iters=100,
                          init_mode="nlm", **kw)
        fg = nb.nlem_denoise_snapshots(noisy, g)[:, rows, :].astype(np.float64)
        o = oracle.make_params(search=21, patch=7, h=h, sigma=sigma, solver=solver, solver_iters=100,
                               init_mode="nlm", **kw)
        fo = np.empty_like(fg)
        for i, r in enumerate(rows):
            _, fr = oracle.nlem_denoise(X, o, rows=(r, r + 1), snapshots=True)
            fo[:, i, :] = fr[:, r, :]
        err = np.abs(fg - fo)
        assert err.max() <= TOL, (solver, err.max(), np.unravel_index(err.argmax(), err.shape))
        for t in range(100):
            assert abs(_psnr(fg[t], c) - _psnr(fo[t], c)) <= PSNR_TOL, (solver, t)


@pytest.mark.parametrize("cfg,k,S", [(0, 5, 11), (2, 7, 21)])
@pytest.mark.parametrize("iters", [10, 30])
def test_irls_tol0_loose(nb, oracle, cfg, k, S, iters):
    """NLEM-IRLS with the reference's own stop rule, tol = 0 (nlem.cpp:45-48, irls.hpp:58: stop
    on the first non-decrease of the surrogate).  The FP32 surrogate stalls a few passes before
    the FP64 one (measured: ~3 passes earlier on average), so the bar is loose:
    the stop pass per pixel (read from the forward-filled frames) within 25 passes, max |d| <=
    0.1 and the 99th percentile <= 0.05 gray levels, |dPSNR| <= 0.01 dB - against the tight
    1e-2 bar of the fixed-count (tol < 0) runs in test_config4_sweep_vs_oracle."""
    from paper_1501_03879_b200 import synth

    clean, noisy = synth.config_image(cfg)
    if cfg == 2:
        clean, noisy = clean[:96, :128], noisy[:96, :128]
    h = synth.reference_h(20.0, k * k)
    g = nb.NlemParams(search=S, patch=k, h=h, sigma=20.0, solver="irls", solver_iters=iters,
                      epsilon=1e-6, irls_tol=0.0)
    o = oracle.make_params(search=S, patch=k, h=h, sigma=20.0, solver="irls", solver_iters=iters,
                           epsilon=1e-6, irls_tol=0.0)
    fg = nb.nlem_denoise_snapshots(noisy, g).astype(np.float64)
    _, fo = oracle.nlem_denoise(noisy.astype(np.float64), o, snapshots=True)

    def stop_pass(f):
        same = np.ones(f.shape[1:], bool)
        st = np.full(f.shape[1:], f.shape[0])
        for t in range(f.shape[0] - 1, 0, -1):
            same &= f[t] == f[t - 1]
            st[same] = t
        return st

    assert np.abs(stop_pass(fg) - stop_pass(fo)).max() <= 25
    d = np.abs(fg[-1] - fo[-1])
    assert d.max() <= 0.1 and np.percentile(d, 99) <= 0.05, (d.max(), np.percentile(d, 99))
    c = clean.astype(np.float64)
    assert abs(_psnr(fg[-1], c) - _psnr(fo[-1], c)) <= PSNR_TOL
