"""Batched IRLS (irls_euclidean_median) on config-1 shapes: time at T = 1, 10, 50 (tol < 0)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1501_03879_b200 as nb
from paper_1501_03879_b200 import synth

B = int(os.environ.get("B", 65536))
pts, w = synth.point_sets(B)
P, W = torch.from_numpy(pts).cuda(), torch.from_numpy(w).cuda()
for T in [int(t) for t in os.environ.get("TS", "1,10,50").split(",")]:
    cfg = nb.IrlsConfig(epsilon=1e-4, max_iter=T, tol=-1.0)
    ts = []
    for i in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        nb.irls_euclidean_median(P, W, cfg)
        b.record(); torch.cuda.synchronize()
        if i: ts.append(a.elapsed_time(b))
    ms = min(ts)
    print(json.dumps({"T": T, "ms": round(ms, 3), "cycles_per_problem_per_SM": round(ms * 1e-3 * 1.965e9 * 148 / B),
                      "frac_alg_5flops": 5 * 49 * 441 * T * B / (ms * 1e-3) / 74.45e12}), flush=True)
