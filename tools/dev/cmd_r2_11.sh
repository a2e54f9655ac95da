cd $GRAFT_REPO_ROOT
timeout 600 python -c "
import sys, os; sys.path.insert(0, 'tools'); import bench_secondary as b
import json; r = b.measure(); print(json.dumps({k: v for k, v in r.items() if k.startswith('config1')}))"
timeout 300 python tools/dev/small_mu.py 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_batched_lr.py tests/test_gpu_parity.py tests/test_gpu_edge.py -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu_b.log 2>&1; tail -4 gpurun_out/pytest_gpu_b.log
