"""Per-sweep slope and per-problem intercept of the batched ADMM kernel (config 1 shapes):
time B problems (n=441, d=49, box [0,255], mu=1) at T = 1, 10, 50."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1501_03879_b200 as nb
from paper_1501_03879_b200 import synth

B = int(os.environ.get("B", 65536))
pts, w = synth.point_sets(B)
P, W = torch.from_numpy(pts).cuda(), torch.from_numpy(w).cuda()
box = nb.BoxConstraint.interval(0.0, 255.0)
for T in [int(t) for t in os.environ.get("TS", "1,10,50").split(",")]:
    cfg = nb.AdmmConfig(mu=1.0, max_iter=T)
    ts = []
    for i in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        nb.admm_euclidean_median(P, W, box, cfg)
        b.record(); torch.cuda.synchronize()
        if i: ts.append(a.elapsed_time(b))
    ms = min(ts)
    cyc = ms * 1e-3 * 1.965e9 * 148 / B
    print(json.dumps({"T": T, "ms": round(ms, 3), "cycles_per_problem_per_SM": round(cyc),
                      "frac_alg": 12 * 49 * 441 * T * B / (ms * 1e-3) / 74.45e12}), flush=True)
