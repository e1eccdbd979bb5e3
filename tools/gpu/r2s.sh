mkdir -p gpurun_out/r2s
timeout 900 python -m pytest tests/test_gpu_parity.py -k "lu or factor_matches or bulk or pipelined" -x -q > gpurun_out/r2s/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2s/pytest.log
for c in "C2" "8192 128" "16384 256" "4096 64"; do echo "== $c"; for cl in 8 16; do timeout 600 python tools/bulk_partition_ab.py $c --reps 3 --sms 0,-1 --lucl $cl; done; done 2>&1 | cut -c1-110
echo "== C3"; timeout 900 python tools/bulk_partition_ab.py C3 --reps 1 --sms 0 --lucl 8 | cut -c1-110
