set -x
mkdir -p gpurun_out/r2c
timeout 900 python -m pytest tests/test_gpu_norms.py tests/test_dist.py tests/test_gpu_parity.py -k "norms or permute_touched or dist or lookahead" -x -q > gpurun_out/r2c/pytest_a.log 2>&1; echo "pytest a rc=$?"; tail -15 gpurun_out/r2c/pytest_a.log
timeout 900 python tools/schedule_ab.py C2 3 > gpurun_out/r2c/ab_c2.txt 2>&1; echo "ab c2 rc=$?"; cat gpurun_out/r2c/ab_c2.txt | grep -v '^{'
timeout 1200 python tools/schedule_ab.py C3 1 > gpurun_out/r2c/ab_c3.txt 2>&1; echo "ab c3 rc=$?"; cat gpurun_out/r2c/ab_c3.txt | grep -v '^{'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c/launches_c2.csv python tools/profile_run.py C2 > gpurun_out/r2c/ncu_c2.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lu_leaf_reg -s 2 -c 1 -o gpurun_out/r2c/lu_leaf_4096 python tools/leaf_probe.py lu 4096 2 > gpurun_out/r2c/ncu_lu.log 2>&1; echo "ncu lu rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lu_panel_kernel -s 2 -c 1 -o gpurun_out/r2c/lu_grid_32768 python tools/leaf_probe.py lu 32768 2 > gpurun_out/r2c/ncu_lu2.log 2>&1; echo "ncu lu2 rc=$?"
for r in 1024 2048 4096 8192 16384 32768 63488; do python tools/leaf_probe.py lu $r 5; done > gpurun_out/r2c/leaf_probe.txt 2>&1
cat gpurun_out/r2c/leaf_probe.txt
