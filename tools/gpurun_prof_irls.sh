cd $GRAFT_REPO_ROOT
TS=1,10,50 timeout 600 python tools/dev/batched_irls.py > gpurun_out/irls_slope2.log 2>&1; cat gpurun_out/irls_slope2.log
timeout 600 python tools/prof_nlem.py --what irls > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:irls_batched_reg -s 1 -c 1 -f \
    -o gpurun_out/prof_irls2_full python tools/prof_nlem.py --what irls > gpurun_out/ncu_irls2.log 2>&1; tail -1 gpurun_out/ncu_irls2.log
