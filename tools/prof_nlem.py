"""Small fixed workload for ncu captures: one NLEM launch on a row band of the config-3
image (same kernel, same per-pixel work as the bench), or a config-1 batch (ADMM or IRLS)."""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1501_03879_b200 as nb
from paper_1501_03879_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--what", default="nlem", choices=["nlem", "admm", "irls"])
ap.add_argument("--rows", type=int, default=32)
ap.add_argument("--problems", type=int, default=2048)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
if a.what == "nlem":
    _, noisy = synth.noisy_image(4096, 4096, 2000, 1500, 30.0)
    p = nb.NlemParams(search=21, patch=7, h=10 * 30.0 * math.sqrt(49), solver_iters=10, mu=1.0,
                      init_mode="nlm")
    X = torch.from_numpy(noisy).cuda()
    r0 = 2048
    for _ in range(a.reps):
        out = nb.nlem_denoise_rows(X[r0 - 13:r0 + a.rows + 13], r0 - 13, 4096, 4096, r0, a.rows, p)
else:
    pts, w = synth.point_sets(a.problems)
    P, W = torch.from_numpy(pts).cuda(), torch.from_numpy(w).cuda()
    for _ in range(a.reps):
        if a.what == "admm":
            r = nb.admm_euclidean_median(P, W, nb.BoxConstraint.interval(0, 255), nb.AdmmConfig(mu=1.0, max_iter=50))
        else:  # the batched IRLS comparator at config-1 shapes, fixed count (tol < 0)
            r = nb.irls_euclidean_median(P, W, nb.IrlsConfig(epsilon=1e-4, max_iter=50, tol=-1.0))
torch.cuda.synchronize()
print("done")
