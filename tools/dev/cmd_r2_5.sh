cd $GRAFT_REPO_ROOT
NLEM_LR_STATS=1 timeout 300 python tools/dev/small_mu.py 2>&1 | tail -12
NLEM_KERNEL=tile timeout 300 python tools/dev/small_mu.py 2>&1 | head -2
timeout 900 python tools/ab_time.py '' lrr1 --reps=8 --rows=512
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -25 gpurun_out/pytest_gpu.log
