mkdir -p gpurun_out/r2o
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q > gpurun_out/r2o/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2o/pytest.log | grep -v "^ "
for c in "C2" "8192 128" "16384 256" "4096 64"; do echo "== $c"; timeout 600 python tools/bulk_partition_ab.py $c --reps 3 --sms 0; timeout 600 python tools/bulk_partition_ab.py $c --reps 3 --sms 0 --no-lula; done > gpurun_out/r2o/ab.txt 2>&1; cut -c1-300 gpurun_out/r2o/ab.txt
