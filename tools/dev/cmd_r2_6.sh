cd $GRAFT_REPO_ROOT
NLEM_LR_STATS=1 timeout 300 python tools/dev/small_mu.py 2>&1 | grep -v "^nlem_lr\|^admm_lr" | tail -6
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -25 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
