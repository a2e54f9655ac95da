"""Secondary measurements (not the driver's headline line): BASELINE config 1 (batched
standalone EM-ADMM, 65,536 problems, n=441, d=49, T=50, box and unconstrained, problems/s)
and config 2 (NLEM 512^2, Mpixels/s), device-resident, CUDA-event timed, L2 flushed.
Prints one JSON object."""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1501_03879_b200 as nb
from paper_1501_03879_b200 import _lib as L, synth

PEAK = 148 * 128 * 2 * 1.965e9 / 1e12


def timed(fn, reps, flush):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def measure(problems=65536, reps=3):
    class A:
        pass
    a = A()
    a.problems, a.reps = problems, reps
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    res = {}
    # ---- config 1
    B, n, d, T = a.problems, 441, 49, 50
    t0 = time.time()
    P = torch.empty((B, n, d), device="cuda")
    W = torch.empty((B, n), device="cuda")
    step = 4096
    for b0 in range(0, B, step):
        nb_ = min(step, B - b0)
        pts, w = synth.point_sets(nb_, first=b0)
        P[b0:b0 + nb_].copy_(torch.from_numpy(pts))
        W[b0:b0 + nb_].copy_(torch.from_numpy(w))
    gen_s = time.time() - t0
    z = torch.empty((B, d), device="cuda")
    cfg = L.AdmmConfigC()
    cfg.mu, cfg.max_iter, cfg.tol_primal = 1.0, T, 0.0
    lib = L.load()
    import ctypes as C
    for name, box in (("box", nb.BoxConstraint.interval(0.0, 255.0)),
                      ("unconstrained", nb.BoxConstraint.unconstrained())):
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)

        def run():
            lib.nlem_admm_batched(C.c_void_p(P.data_ptr()), C.c_void_p(W.data_ptr()), B, n, d, None,
                                  box.c(), cfg, C.c_void_p(z.data_ptr()), None, None, None, None,
                                  None, st)
        ms = timed(run, a.reps, flush)
        flops = 12 * d * T * n * B
        res[f"config1_{name}"] = {"problems_per_s": B / (ms / 1e3), "ms": ms,
                                  "tflops_algorithmic": flops / (ms / 1e3) / 1e12,
                                  "frac_fp32_peak": flops / (ms / 1e3) / 1e12 / PEAK}
    # the IRLS surrogate solver (irls.hpp:21-68) on the same point sets: eps = 1e-4, T = 50
    # sweeps at a fixed count (tol < 0); algorithmic work 5 d per point and sweep
    icfg = L.IrlsConfigC()
    icfg.epsilon, icfg.max_iter, icfg.tol = 1e-4, T, -1.0

    def run_irls():
        lib.nlem_irls_batched(C.c_void_p(P.data_ptr()), C.c_void_p(W.data_ptr()), B, n, d, None,
                              icfg, C.c_void_p(z.data_ptr()), None, None, None, None,
                              C.c_void_p(torch.cuda.current_stream().cuda_stream))
    ms = timed(run_irls, a.reps, flush)
    flops = 5 * d * T * n * B
    res["config1_irls"] = {"problems_per_s": B / (ms / 1e3), "ms": ms,
                           "tflops_algorithmic": flops / (ms / 1e3) / 1e12,
                           "frac_fp32_peak": flops / (ms / 1e3) / 1e12 / PEAK}
    res["config1_generation_s"] = gen_s
    # small-mu regime: the reference's default mu = 1e-3 (types.hpp:121) at T = 10 on the same point
    # sets - the prox scales saturate, the probe routes the batch to the exact p-form kernel
    # (no slower than that kernel alone)
    cfg_s = L.AdmmConfigC()
    cfg_s.mu, cfg_s.max_iter, cfg_s.tol_primal = 1e-3, 10, 0.0
    box = nb.BoxConstraint.interval(0.0, 255.0)

    def run_small():
        lib.nlem_admm_batched(C.c_void_p(P.data_ptr()), C.c_void_p(W.data_ptr()), B, n, d, None,
                              box.c(), cfg_s, C.c_void_p(z.data_ptr()), None, None, None, None,
                              None, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    ms = timed(run_small, a.reps, flush)
    res["config1_small_mu"] = {"mu": 1e-3, "iters": 10, "problems_per_s": B / (ms / 1e3), "ms": ms,
                               "path": "small_mu_probe_kernel -> exact p-form kernel (admm_batched_fast)"}
    del P, W
    # config-3 band (512 rows x 4096) at mu = 1e-3, T = 10: probe -> ring-12 build of the low-rank
    # kernel (T <= 12; the exact tile kernel beyond)
    _, noisy3 = synth.noisy_image(4096, 4096, 2000, 1500, 30.0)
    rows3, r0 = 512, 1024
    band = torch.from_numpy(noisy3[r0 - 13:r0 + rows3 + 13]).cuda()
    for key, mu in (("config3_band_mu1", 1.0), ("config3_band_small_mu", 1e-3)):
        p3 = nb.NlemParams(search=21, patch=7, h=10 * 30.0 * math.sqrt(49), sigma=30.0, solver_iters=10,
                           mu=mu, init_mode="nlm")
        ms = timed(lambda: nb.nlem_denoise_rows(band, r0 - 13, 4096, 4096, r0, rows3, p3), a.reps, flush)
        res[key] = {"mu": mu, "rows": rows3, "mpix_per_s": rows3 * 4096 / (ms / 1e3) / 1e6, "ms": ms}
    # the reference's default NlemParams (nlem.hpp:23-35: 4 sweeps, mu = 1e-3, noisy-patch init)
    # with the reference CLI's h = 10 sigma: 4 sweeps fit the history ring, so the low-rank kernel
    # runs the saturated regime itself (tests/test_gpu_parity.py::test_reference_default_params_in_lr_kernel)
    p3d = nb.NlemParams(search=21, patch=7, h=10 * 30.0, sigma=30.0, solver_iters=4, mu=1e-3,
                        init_mode="noisy")
    ms = timed(lambda: nb.nlem_denoise_rows(band, r0 - 13, 4096, 4096, r0, rows3, p3d), a.reps, flush)
    res["config3_band_reference_defaults"] = {"iters": 4, "mu": 1e-3, "init": "noisy", "rows": rows3,
                                              "mpix_per_s": rows3 * 4096 / (ms / 1e3) / 1e6, "ms": ms}
    # the NLM baseline (nlm.cpp:31-51) on the same band: NlmOnly mode of the low-rank kernel
    p3n = nb.NlemParams(search=21, patch=7, h=10 * 30.0 * math.sqrt(49), sigma=30.0, solver="nlm_only",
                        solver_iters=10, mu=1.0, init_mode="nlm")
    ms = timed(lambda: nb.nlem_denoise_rows(band, r0 - 13, 4096, 4096, r0, rows3, p3n), a.reps, flush)
    res["config3_band_nlm_only"] = {"rows": rows3, "mpix_per_s": rows3 * 4096 / (ms / 1e3) / 1e6, "ms": ms}
    del band
    # ---- config 2
    clean, noisy = synth.config_image(2)
    p = nb.NlemParams(search=21, patch=7, h=10 * 20.0 * math.sqrt(49), sigma=20.0, solver_iters=10,
                      mu=1.0, init_mode="nlm")
    X = torch.from_numpy(noisy).cuda()
    ms = timed(lambda: nb.nlem_denoise(X, p), a.reps, flush)
    res["config2"] = {"mpix_per_s": 512 * 512 / (ms / 1e3) / 1e6, "ms": ms}
    # ---- config 4: convergence sweep, ADMM vs IRLS (eps=1e-4, fixed count), T = 1..100
    sweep = {}
    for sigma in (10.0, 20.0, 40.0, 60.0):
        clean, noisy = synth.noisy_image(512, 512, 40, 30, sigma)
        X = torch.from_numpy(noisy).cuda()
        h = 10 * sigma * math.sqrt(49)
        entry = {}
        for solver, kw in (("admm", dict(mu=1.0)), ("irls", dict(epsilon=1e-4, irls_tol=-1.0))):
            pr = nb.NlemParams(search=21, patch=7, h=h, sigma=sigma, solver=solver, solver_iters=100,
                               init_mode="nlm", **kw)
            ms = timed(lambda: nb.nlem_denoise_snapshots(X, pr), 1, flush)
            fr = nb.nlem_denoise_snapshots(X, pr).cpu().numpy().astype(np.float64)
            mse = ((fr - clean.astype(np.float64)[None]) ** 2).mean(axis=(1, 2))
            psnr = 10 * np.log10(255.0 ** 2 / mse)
            entry[solver] = {"ms_per_iteration": ms / 100,
                             "psnr_db": {str(t): float(psnr[t - 1]) for t in (1, 2, 3, 4, 5, 10, 20, 50, 100)}}
        entry["psnr_noisy_db"] = float(10 * np.log10(255.0 ** 2 / ((noisy.astype(np.float64) - clean) ** 2).mean()))
        sweep[str(int(sigma))] = entry
    res["config4"] = sweep
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problems", type=int, default=65536)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    print(json.dumps(measure(a.problems, a.reps)))


if __name__ == "__main__":
    main()
