# Round-2 measurement pass (one gpurun call): FP32 peak microbenchmark, the bench line, the
# bench's kernel launch list under ncu, and one ncu --set full capture of nlem_pixels_lr.
cd $GRAFT_REPO_ROOT
python -c 'from paper_1501_03879_b200 import build as B; B.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
./tools/fp32_peak > gpurun_out/fp32_peak.txt 2>&1; cat gpurun_out/fp32_peak.txt
timeout 1500 python bench.py > gpurun_out/bench_r2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r2.log | cut -c1-400
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 600 python tools/prof_nlem.py --what nlem --rows 64 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nlem_pixels_lr -s 1 -c 1 -f \
  -o gpurun_out/r2_lr_full python tools/prof_nlem.py --what nlem --rows 64 > gpurun_out/ncu_lr_full.log 2>&1; echo "ncu full rc=$?"
