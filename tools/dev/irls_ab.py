"""A/B of the batched kernels between two library builds (NLEM_LIB_VARIANT) on config-1 shapes
(65,536 x n=441 x d=49, T=50): IRLS (eps=1e-4, tol<0 and tol=0) and ADMM (mu=1, box [0,255]);
median ms of 7 launches (CUDA events, L2 flushed) and a bitwise comparison of the outputs
(minimiser, objective, iterations).  usage (GPU box): python tools/dev/irls_ab.py old ''"""
import json, os, subprocess, sys

CHILD = r"""
import ctypes as C, json, sys, numpy as np, torch
sys.path.insert(0, %(root)r)
import paper_1501_03879_b200 as nb
from paper_1501_03879_b200 import _lib as L, synth
B, n, d, T = 65536, 441, 49, 50
P = torch.empty((B, n, d), device="cuda"); W = torch.empty((B, n), device="cuda")
for b0 in range(0, B, 8192):
    pts, w = synth.point_sets(8192, first=b0)
    P[b0:b0 + 8192].copy_(torch.from_numpy(pts)); W[b0:b0 + 8192].copy_(torch.from_numpy(w))
z = torch.empty((B, d), device="cuda"); obj = torch.empty(B, device="cuda")
it = torch.empty(B, dtype=torch.int32, device="cuda")
icfg = L.IrlsConfigC(); icfg.epsilon, icfg.max_iter, icfg.tol = 1e-4, T, (0.0 if %(tol)r == "admm" else %(tol)r)
lib = L.load(); flush = torch.empty(64 << 20, device="cuda")
box = nb.BoxConstraint.interval(0.0, 255.0)
acfg = L.AdmmConfigC(); acfg.mu, acfg.max_iter, acfg.tol_primal = 1.0, T, 0.0
def run():
    if %(tol)r == "admm":
        lib.nlem_admm_batched(C.c_void_p(P.data_ptr()), C.c_void_p(W.data_ptr()), B, n, d, None, box.c(), acfg,
                              C.c_void_p(z.data_ptr()), C.c_void_p(obj.data_ptr()), C.c_void_p(it.data_ptr()),
                              None, None, None, C.c_void_p(torch.cuda.current_stream().cuda_stream))
        return
    lib.nlem_irls_batched(C.c_void_p(P.data_ptr()), C.c_void_p(W.data_ptr()), B, n, d, None, icfg,
                          C.c_void_p(z.data_ptr()), C.c_void_p(obj.data_ptr()), C.c_void_p(it.data_ptr()),
                          None, None, C.c_void_p(torch.cuda.current_stream().cuda_stream))
run(); torch.cuda.synchronize(); ts = []
for _ in range(%(reps)d):
    flush.fill_(1.0)
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); run(); e.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(e))
np.save(%(out)r, np.concatenate([z.cpu().numpy().ravel(), obj.cpu().numpy(), it.cpu().numpy().astype(np.float32)]))
print(json.dumps({"ms_med": float(np.median(ts)), "ms_min": min(ts)}))
"""

root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
res = {}
for tol in (-1.0, 0.0, "admm"):
    for v in sys.argv[1:]:
        out = f"/tmp/irls_{v or 'cur'}_{tol}.npy"
        env = dict(os.environ, NLEM_LIB_VARIANT=v)
        r = subprocess.run([sys.executable, "-c", CHILD % dict(root=root, reps=7, out=out, tol=tol)],
                           env=env, capture_output=True, text=True)
        res[f"{v or 'cur'} tol={tol}"] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-800:]
    import numpy as np
    outs = [np.load(f"/tmp/irls_{v or 'cur'}_{tol}.npy") for v in sys.argv[1:]]
    res[f"bitwise_equal tol={tol}"] = all(np.array_equal(outs[0], o) for o in outs[1:])
print(json.dumps(res, indent=1))
