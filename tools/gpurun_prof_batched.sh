# ncu --set full of the two batched kernels at config-1 shapes (one launch each, 2,048 problems),
# plus the IRLS iteration slope.  Each ncu pass runs after its command exited 0 without ncu.
cd $GRAFT_REPO_ROOT
TS=1,10,50 timeout 600 python tools/dev/batched_irls.py > gpurun_out/irls_slope.log 2>&1; cat gpurun_out/irls_slope.log
for w in irls admm; do
  k=$([ $w = irls ] && echo irls_batched_reg || echo admm_batched_lr)
  timeout 600 python tools/prof_nlem.py --what $w > gpurun_out/prof_plain_$w.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -f \
    -o gpurun_out/prof_${w}_full python tools/prof_nlem.py --what $w > gpurun_out/ncu_${w}_full.log 2>&1
  tail -1 gpurun_out/ncu_${w}_full.log
done
true
