"""A/B timing of NLEM kernel build variants on a row band of the config-3 image.

usage (on the GPU box): python tools/ab_time.py '' xw4 ...
Each variant runs in its own process (NLEM_LIB_VARIANT selects _lib/libnlem_b200_<v>.so) and
reports min / median / max milliseconds over --reps launches of the same band (CUDA events),
so step-to-step noise of the full bench does not decide an A/B.
"""
import json
import os
import subprocess
import sys

CHILD = r"""
import json, math, sys, torch
sys.path.insert(0, %(root)r)
import paper_1501_03879_b200 as nb
from paper_1501_03879_b200 import synth
_, noisy = synth.noisy_image(4096, 4096, 2000, 1500, 30.0)
p = nb.NlemParams(search=21, patch=7, h=10 * 30.0 * math.sqrt(49), solver_iters=10, mu=1.0,
                  init_mode="nlm")
X = torch.from_numpy(noisy).cuda()
rows, r0 = %(rows)d, 1024
band = X[r0 - 13:r0 + rows + 13].contiguous()
ts = []
for i in range(%(reps)d + 2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    out = nb.nlem_denoise_rows(band, r0 - 13, 4096, 4096, r0, rows, p)
    b.record()
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(a.elapsed_time(b))
ts.sort()
print(json.dumps({"min": ts[0], "med": ts[len(ts) // 2], "max": ts[-1],
                  "mpix_s": rows * 4096 / ts[0] / 1e3, "sum": float(out.double().sum())}))
"""


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    reps = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--reps=")), 12))
    rows = int(next((a.split("=")[1] for a in sys.argv if a.startswith("--rows=")), 256))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for rnd in range(2):  # two interleaved rounds: drift shows up as round-to-round change
        for v in args or [""]:
            # "variant" or "variant:ENV=VALUE" (e.g. ":NLEM_NO_TMA=1" = production with TMA off)
            lib_v, _, envs = v.partition(":")
            env = dict(os.environ, NLEM_LIB_VARIANT=lib_v)
            if envs:
                k, _, val = envs.partition("=")
                env[k] = val
            r = subprocess.run([sys.executable, "-c", CHILD % dict(root=root, reps=reps, rows=rows)],
                               env=env, capture_output=True, text=True, timeout=900)
            line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
            print(f"round {rnd} variant {v or 'prod':6s} {line}", flush=True)


if __name__ == "__main__":
    main()
