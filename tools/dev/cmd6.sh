cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider -k "lr_" > gpurun_out/pytest_gpu_lr.log 2>&1; tail -15 gpurun_out/pytest_gpu_lr.log
