# A/B the NLEM kernels on the bench workload (device-resident value only)
cd $GRAFT_REPO_ROOT
for k in seg2 tile; do
  echo "== $k"; NLEM_KERNEL=$k timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
done
