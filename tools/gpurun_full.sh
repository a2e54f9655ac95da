# Round evidence in one box call: full default bench line, the ncu launch list of the same
# command (gpu__time_duration per launch), and an ncu --set full capture of the NLEM tile kernel
# (source-level, for profiles/).  Each ncu pass runs only after its command exited 0 without ncu.
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
nproc
timeout 1500 python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log | cut -c1-400
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/bench_small.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_launches.log 2>&1
tail -2 gpurun_out/ncu_launches.log
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:nlem_pixels_lr -c 1 --csv --log-file gpurun_out/dram_bench_launch.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-secondary > gpurun_out/ncu_dram.log 2>&1
tail -1 gpurun_out/ncu_dram.log
timeout 600 python tools/prof_nlem.py --what nlem > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nlem_pixels_lr -s 1 -c 1 -f \
  -o gpurun_out/prof_lr_full python tools/prof_nlem.py --what nlem > gpurun_out/ncu_lr_full.log 2>&1
tail -2 gpurun_out/ncu_lr_full.log
true
