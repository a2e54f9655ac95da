cd $GRAFT_REPO_ROOT
timeout 300 python tools/prof_nlem.py --what nlem > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nlem_pixels_lr -s 1 -c 1 -f \
  -o gpurun_out/prof_lr7 python tools/prof_nlem.py --what nlem > gpurun_out/ncu_lr.log 2>&1
tail -1 gpurun_out/ncu_lr.log
