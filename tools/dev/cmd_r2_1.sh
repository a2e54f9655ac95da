cd $GRAFT_REPO_ROOT
python -c 'from paper_1501_03879_b200 import build as B; B.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -5 gpurun_out/build.log; exit 1; }
NLEM_LR_STATS=1 timeout 300 python tools/dev/small_mu.py 2>&1 | grep -v "^nlem_lr" | tail -4
NLEM_LR_STATS=1 timeout 300 python tools/dev/small_mu.py 2>&1 | grep "^nlem_lr" | sort | uniq -c
NLEM_KERNEL=tile timeout 300 python tools/dev/small_mu.py 2>&1 | tail -2
timeout 300 python tools/ab_time.py --reps=8
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
