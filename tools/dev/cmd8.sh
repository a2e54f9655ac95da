cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python -c "
import sys, json; sys.path.insert(0, 'tools'); import bench_secondary as b
r = b.measure(); print(json.dumps({k: r[k] for k in r if k.startswith('config4') or k=='config2'})[:3000])"
