cd $GRAFT_REPO_ROOT
NLEM_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2.log 2>&1; echo "rc=$?"; grep metric gpurun_out/bench_n2.log | cut -c1-400; tail -3 gpurun_out/bench_n2.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-600
