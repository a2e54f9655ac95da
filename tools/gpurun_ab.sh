# A/B build variants on the bench workload (device-resident value + e2e), then GPU parity for each.
# usage (on the box): VARIANTS="'' xw1" bash tools/gpurun_ab.sh
cd $GRAFT_REPO_ROOT
for v in ${VARIANTS:-""}; do
  v=${v//\'/}
  echo "== variant '${v}'"
  NLEM_LIB_VARIANT=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ab_$v.log 2>&1 || tail -5 gpurun_out/ab_$v.log
  tail -1 gpurun_out/ab_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'])" || echo "bench failed"
done
for v in ${VARIANTS:-""}; do
  v=${v//\'/}
  echo "== tests variant '${v}'"
  NLEM_LIB_VARIANT=$v timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -3
done
