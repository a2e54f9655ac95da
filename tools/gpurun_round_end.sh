cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_full.log | cut -c1-300
bash tools/gpurun_multirank.sh
