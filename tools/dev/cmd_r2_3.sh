cd $GRAFT_REPO_ROOT
timeout 900 python tools/ab_time.py '' nocancel_nosat_nobrk --reps=8 --rows=512
NLEM_LR_STATS=1 timeout 300 python tools/dev/small_mu.py 2>&1 | tail -6
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -25 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
