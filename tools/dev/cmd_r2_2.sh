cd $GRAFT_REPO_ROOT
timeout 900 python tools/ab_time.py '' nocancel nosat nobrk nocancel_nosat_nobrk --reps=8 --rows=512
