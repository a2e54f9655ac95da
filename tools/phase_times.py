"""Per-phase cycle counts of the NLEM tile kernel sweep (debug build with NLEM_PHASE_PROFILE).
usage: python tools/phase_times.py   (builds _lib/libnlem_b200_prof.so first)"""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1501_03879_b200 import build as B

_var = os.environ.get("PROF_VARIANT", "prof")
so = B.variant_path(_var)
if not os.path.exists(so):  # prebuilt here and shipped, or built on the box
    so = B.build(force=True, variant=_var)
import paper_1501_03879_b200._lib as L

L.SO_PATH = so
import paper_1501_03879_b200 as nb
import torch
from paper_1501_03879_b200 import synth

_, noisy = synth.noisy_image(512, 512, 40, 30, 30.0)
p = nb.NlemParams(search=21, patch=7, h=10 * 30.0 * math.sqrt(49), solver_iters=10, mu=1.0,
                  init_mode="nlm")
X = torch.from_numpy(noisy).cuda()
out = nb.nlem_denoise_rows(X[200:280], 200, 512, 512, 213, 16, p)
torch.cuda.synchronize()
buf = np.zeros((2, 64, 16), np.int64)
lib = L.load(build_if_missing=False)
assert lib.nlem_debug_phase_times(buf.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
names = ["update+norm", "norm-exchange", "s+bcast", "g+flags", "barrier+consensus+barrier", "->next",
         "  red write+barrier1", "  consensus loads+tree", "  xor shuffles", "  (cluster xchg)+finish", "  barrier2",
         "  cluster exchange only"]
for w in range(2):
    d = buf[w]
    valid = [i for i in range(64) if d[i, 0] and d[i, 5]]
    rows = []
    for i in valid:
        seg = [d[i, k + 1] - d[i, k] for k in range(5)]
        nxt = d[i + 1, 0] - d[i, 5] if i + 1 in valid else 0
        sub = [d[i, 6] - d[i, 4], d[i, 7] - d[i, 6], d[i, 8] - d[i, 7], d[i, 9] - d[i, 8],
               d[i, 10] - d[i, 9], d[i, 11] - d[i, 8]]
        rows.append(seg + [nxt] + sub)
    a = np.array(rows[2:])  # skip warm-up sweeps
    print(f"warp {'0' if w == 0 else 'last'}: sweeps={len(a)}")
    if len(a) == 0:
        continue
    for k, n in enumerate(names):
        print(f"   {n:28s} mean {a[:, k].mean():8.1f}  median {np.median(a[:, k]):8.1f}")
    print(f"   total per sweep (median)     {np.median(a[:, :5].sum(1) + a[:, 5]):8.1f}")

wb = np.zeros((32, 64, 4), np.int64)
assert lib.nlem_debug_warp_times(wb.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
nw = 16
rows = []
for it in range(4, 60):
    st = wb[:nw, it, 0]
    if (st == 0).any() or (wb[:nw, it + 1, 0] == 0).any():
        continue
    t0 = st.min()
    rows.append([st - t0, wb[:nw, it, 1] - t0, wb[:nw, it, 2] - t0, wb[:nw, it, 3] - t0,
                 wb[:nw, it + 1, 0] - t0])
a = np.array(rows)  # [sweeps, 5, warps]
med = np.median(a, axis=0)
print("per-warp median cycles since the earliest sweep start (sweep start, red written, after B1, after B2, next start):")
for w in range(nw):
    print(f"  warp {w:2d}: " + "  ".join(f"{x:7.0f}" for x in med[:, w]))

sb = np.zeros((64, 8), np.int64)
if hasattr(lib, "nlem_debug_setup_times") and lib.nlem_debug_setup_times(
        sb.ctypes.data_as(C.POINTER(C.c_longlong))) == 0:
    segs = ["tile wait+neq scan", "syncthreads_or", "weights+bcast", "init consensus", "prefetch issue",
            "sweeps", "epilogue->next pixel"]
    rows = []
    for i in range(2, 62):
        d = sb[i]
        if (d[:7] == 0).any() or sb[i + 1, 0] == 0:
            continue
        rows.append([d[k + 1] - d[k] for k in range(6)] + [sb[i + 1, 0] - d[6]])
    if rows:
        a = np.array(rows)
        print(f"per-pixel setup (thread 0, CTA 0; {len(a)} pixels), median cycles:")
        for k, n in enumerate(segs):
            print(f"   {n:24s} {np.median(a[:, k]):8.0f}")
        print(f"   {'total per pixel':24s} {np.median(a.sum(1)):8.0f}")
