cd $GRAFT_REPO_ROOT
timeout 900 python tools/ab_time.py '' lrr1 --reps=8 --rows=512
timeout 1500 python -m pytest tests/test_gpu_edge.py tests/test_gpu_nlm_patch.py tests/test_gpu_configs.py -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu_new.log 2>&1; tail -30 gpurun_out/pytest_gpu_new.log
