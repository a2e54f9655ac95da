"""Per-sweep slope and setup intercept of an NLEM kernel: time a config-3 band at T = 1, 5, 10, 20."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1501_03879_b200 as nb
from paper_1501_03879_b200 import synth
_, noisy = synth.noisy_image(4096, 4096, 2000, 1500, 30.0)
X = torch.from_numpy(noisy).cuda()
rows, r0 = int(os.environ.get("ROWS", 128)), 1024
band = X[r0 - 13:r0 + rows + 13].contiguous()
for T in (1, 5, 10, 20):
    p = nb.NlemParams(search=21, patch=7, h=10 * 30.0 * math.sqrt(49), solver_iters=T, mu=1.0, init_mode="nlm")
    ts = []
    for i in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        nb.nlem_denoise_rows(band, r0 - 13, 4096, 4096, r0, rows, p)
        b.record(); torch.cuda.synchronize()
        if i: ts.append(a.elapsed_time(b))
    ms = min(ts)
    cyc_px = ms * 1e-3 * 1.965e9 * 148 / (rows * 4096)
    print(json.dumps({"T": T, "ms": round(ms, 3), "cycles_per_pixel_per_SM": round(cyc_px)}), flush=True)
