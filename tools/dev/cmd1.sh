cd $GRAFT_REPO_ROOT
timeout 300 python tools/ab_time.py ':NLEM_KERNEL=tile' ':NLEM_KERNEL=lr' --reps=5 > gpurun_out/ab1.log 2>&1; cat gpurun_out/ab1.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -30 gpurun_out/pytest_gpu.log
