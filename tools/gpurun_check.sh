set -x
cd $GRAFT_REPO_ROOT
python -c 'from paper_1501_03879_b200 import build as B; B.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -5 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -40 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -5 gpurun_out/smoke.log
[ "$BENCH" = "1" ] && (timeout 1500 python bench.py --steps 2 --warmup 1 --cpu-sample-rows 2 > gpurun_out/bench.log 2>&1; tail -5 gpurun_out/bench.log)
true
