set -x
mkdir -p gpurun_out/r2i
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q > gpurun_out/r2i/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2i/pytest.log
for r in 1024 4096 8192 16384; do python tools/leaf_probe.py lu $r 5; done > gpurun_out/r2i/leaf_probe.txt 2>&1; python tools/leaf_probe.py qr 2048 5 >> gpurun_out/r2i/leaf_probe.txt 2>&1; cat gpurun_out/r2i/leaf_probe.txt
timeout 600 python tools/schedule_ab.py C2 3 > gpurun_out/r2i/ab_c2.txt 2>&1; grep -v '^{' gpurun_out/r2i/ab_c2.txt | head -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i/launches_c2.csv python tools/profile_run.py C2 > gpurun_out/r2i/ncu_c2.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lu_leaf_fast -s 2 -c 1 -o gpurun_out/r2i/lu_fast_4096 python tools/leaf_probe.py lu 4096 2 > gpurun_out/r2i/ncu_lu.log 2>&1; echo "ncu lu rc=$?"
