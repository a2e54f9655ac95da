cd $GRAFT_REPO_ROOT
timeout 900 python tools/ab_time.py '' np1 lrnp1 --reps=8 --rows=512
