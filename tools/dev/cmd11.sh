cd $GRAFT_REPO_ROOT
timeout 900 python tools/ab_time.py ':NLEM_KERNEL=lr' 'ud7:NLEM_KERNEL=lr' 'ug4:NLEM_KERNEL=lr' 'ud7_ug4:NLEM_KERNEL=lr' --reps=5 > gpurun_out/ab.log 2>&1; cat gpurun_out/ab.log | cut -c1-140
