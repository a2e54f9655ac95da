# ncu --set full of the production image kernel (nlem_pixels_lr) on a config-3 row band.
cd $GRAFT_REPO_ROOT
timeout 600 python tools/prof_nlem.py --what nlem > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nlem_pixels_lr -s 1 -c 1 -f \
  -o gpurun_out/prof_lr_full python tools/prof_nlem.py --what nlem > gpurun_out/ncu_lr_full.log 2>&1
tail -1 gpurun_out/ncu_lr_full.log
