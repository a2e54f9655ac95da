cd $GRAFT_REPO_ROOT
timeout 900 python tools/ab_time.py '' np1 lrnp1 --reps=8 --rows=512
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_nlm_patch.py -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu_lr.log 2>&1; tail -15 gpurun_out/pytest_gpu_lr.log
