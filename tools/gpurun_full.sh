# full bench line + ncu launch list of the same command + compute-sanitizer memcheck (small)
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
nproc
timeout 1500 python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/bench_small.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_launches.log 2>&1
tail -2 gpurun_out/ncu_launches.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch, math
import paper_1501_03879_b200 as nb
from paper_1501_03879_b200 import synth
c, n = synth.noisy_image(40, 37, 6, 4, 20.0)
for (S,k) in ((21,7),(11,5),(7,3),(9,5)):
    p = nb.NlemParams(search=S, patch=k, h=200.0, solver_iters=3, mu=1.0, init_mode='nlm')
    nb.nlem_denoise(n, p); nb.nlem_denoise_snapshots(n, p)
pts, w = synth.point_sets(8)
nb.admm_euclidean_median(pts, w, nb.BoxConstraint.interval(0,255), nb.AdmmConfig(mu=1.0, max_iter=5))
nb.admm_euclidean_median(pts[:, :100, :25].copy(), w[:, :100].copy(), None, nb.AdmmConfig(mu=1.0, max_iter=5))
nb.irls_euclidean_median(pts, w, nb.IrlsConfig(max_iter=5))
print('memcheck workload done')
" > gpurun_out/memcheck.log 2>&1; tail -4 gpurun_out/memcheck.log
true
