cd $GRAFT_REPO_ROOT
timeout 600 python tools/ab_time.py ':NLEM_KERNEL=lr' 'st4:NLEM_KERNEL=lr' --reps=5 > gpurun_out/ab.log 2>&1; cat gpurun_out/ab.log
