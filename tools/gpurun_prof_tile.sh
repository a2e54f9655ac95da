cd $GRAFT_REPO_ROOT
timeout 600 python tools/prof_nlem.py --what nlem > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nlem_pixels_tile -s 1 -c 1 -f -o gpurun_out/prof_tile python tools/prof_nlem.py --what nlem > gpurun_out/ncu_tile.log 2>&1
tail -3 gpurun_out/ncu_tile.log
