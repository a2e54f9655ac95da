cd $GRAFT_REPO_ROOT
timeout 600 python tools/ab_time.py 'base:NLEM_KERNEL=lr' ':NLEM_KERNEL=lr' --reps=5 > gpurun_out/ab.log 2>&1; cat gpurun_out/ab.log
NLEM_KERNEL=lr timeout 300 python tools/dev/lr_iters.py
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
