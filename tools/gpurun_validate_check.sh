cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "validation" --timeout 600 -p no:cacheprovider 2>&1 | tail -3
TS=50 timeout 600 python tools/dev/batched_irls.py 2>&1 | tail -1
python - <<'PY'
import torch, time, json, sys
sys.path.insert(0, '.')
import paper_1501_03879_b200 as nb
from paper_1501_03879_b200 import synth
pts, w = synth.point_sets(65536)
P, W = torch.from_numpy(pts).cuda(), torch.from_numpy(w).cuda()
for name, fn in (("admm_box", lambda: nb.admm_euclidean_median(P, W, nb.BoxConstraint.interval(0, 255), nb.AdmmConfig(mu=1.0, max_iter=50))),):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(json.dumps({name + "_api_ms": min(ts)}))
PY
