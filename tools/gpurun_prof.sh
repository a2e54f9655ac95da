set -x
cd $GRAFT_REPO_ROOT
python -c "import paper_1501_03879_b200._lib as L; L.load()"
timeout 600 python tools/prof_nlem.py --what nlem > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nlem_pixels_tile -s 1 -c 1 -f -o gpurun_out/prof_nlem python tools/prof_nlem.py --what nlem > gpurun_out/ncu_nlem.log 2>&1
tail -3 gpurun_out/ncu_nlem.log
timeout 600 python tools/prof_nlem.py --what admm > gpurun_out/prof_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:admm_batched_fast -s 1 -c 1 -f -o gpurun_out/prof_admm python tools/prof_nlem.py --what admm > gpurun_out/ncu_admm.log 2>&1
tail -3 gpurun_out/ncu_admm.log
true
