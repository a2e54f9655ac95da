cd $GRAFT_REPO_ROOT
timeout 300 python tools/dev/small_mu.py 2>&1 | tail -4
timeout 2400 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_edge.py tests/test_dist_gloo.py -m gpu -q -s --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu_acc.log 2>&1; tail -25 gpurun_out/pytest_gpu_acc.log
