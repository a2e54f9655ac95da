"""Config-3 image at mu = 1 (BASELINE) and mu = 1e-3 (reference default, types.hpp:121), T = 10:
time of the production dispatch (low-rank kernel + hand-off) per 512-row band and the number of
handed-off pixels; with NLEM_KERNEL=tile in the environment the exact tile kernel alone."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1501_03879_b200 as nb
from paper_1501_03879_b200 import synth

_, noisy = synth.noisy_image(4096, 4096, 2000, 1500, 30.0)
X = torch.from_numpy(noisy).cuda()
rows = int(os.environ.get("ROWS", "512"))
r0 = 1024
band = X[r0 - 13:r0 + rows + 13].contiguous()
for mu in (1.0, 1e-3):
    p = nb.NlemParams(search=21, patch=7, h=10 * 30.0 * math.sqrt(49), solver_iters=10, mu=mu,
                      init_mode="nlm")
    ts = []
    for i in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = nb.nlem_denoise_rows(band, r0 - 13, 4096, 4096, r0, rows, p)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = min(ts[1:])
    print(f"kernel={os.environ.get('NLEM_KERNEL', 'prod')} mu={mu} rows={rows}: {t:.2f} ms "
          f"= {rows * 4096 / t / 1e3:.2f} Mpix/s sum={float(out.double().sum()):.6f}", flush=True)

# config 1 (batched standalone solves, n = 441, d = 49, T = 50) at mu = 1 and mu = 1e-3
import numpy as np  # noqa: E402

B = 16384
pts, w = synth.point_sets(B)
P, Wt = torch.from_numpy(pts).cuda(), torch.from_numpy(w).cuda()
for mu in (1.0, 1e-3):
    cfg = nb.AdmmConfig(mu=mu, max_iter=50)
    box = nb.BoxConstraint.interval(0.0, 255.0)
    ts = []
    for i in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        r = nb.admm_euclidean_median(P, Wt, box, cfg)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = min(ts[1:])
    print(f"config1 mu={mu} B={B}: {t:.2f} ms = {B / t / 1e3:.3f} M problems/s", flush=True)
print(f"(NLEM_BATCHED_KERNEL={os.environ.get('NLEM_BATCHED_KERNEL', 'default')})")
