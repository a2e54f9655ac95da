# ncu --set full of the NLEM tile kernel for one build variant: VARIANT=xw4 bash tools/gpurun_prof_variant.sh
cd $GRAFT_REPO_ROOT
export NLEM_LIB_VARIANT=${VARIANT:-}
timeout 600 python tools/prof_nlem.py --what nlem > gpurun_out/prof_plain_${VARIANT}.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nlem_pixels_tile -s 1 -c 1 -f -o gpurun_out/prof_tile_${VARIANT} python tools/prof_nlem.py --what nlem > gpurun_out/ncu_tile_${VARIANT}.log 2>&1
tail -2 gpurun_out/ncu_tile_${VARIANT}.log
