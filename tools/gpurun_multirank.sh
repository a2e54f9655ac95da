# N>1 bench path on a one-GPU box: NLEM_BENCH_SHARE_GPU=1 puts every rank on cuda:0 with gloo
# (timings meaningless; checks the band split, the gather, the band-boundary parity rows and
# the single JSON line), then the reference arm.
cd $GRAFT_REPO_ROOT
for n in 2 4 8; do
  NLEM_BENCH_SHARE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 1 --warmup 3 --no-secondary \
    > gpurun_out/bench_n$n.log 2>&1; echo "n=$n rc=$?"
  grep '"metric"' gpurun_out/bench_n$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('parity', d['parity'])"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-300
