mkdir -p gpurun_out/r2z
timeout 600 python -m pytest tests/test_gpu_parity.py -k "factor_matches or bulk" -x -q > gpurun_out/r2z/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2z/pytest.log
for c in "C2" "8192 256" "16384 256" "4096 256"; do echo "== $c"; for L in 0 16 32 64; do timeout 600 python tools/bulk_partition_ab.py $c --reps 3 --sms 0 --lat-ctas $L; done; done 2>&1 | cut -c1-200
echo "== C3"; for L in 0 32; do timeout 900 python tools/bulk_partition_ab.py C3 --reps 1 --sms 0 --lat-ctas $L | cut -c1-200; done
