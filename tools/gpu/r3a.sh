mkdir -p gpurun_out/r3a
timeout 900 python -m pytest tests/test_gpu_parity.py -k "merge_stream or pipelined or factor_matches" -x -q > gpurun_out/r3a/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r3a/pytest.log
for c in "C2" "8192 256" "16384 256" "4096 256" "2048 256"; do echo "== $c"; timeout 600 python tools/bulk_partition_ab.py $c --reps 3 --sms 0; timeout 600 python tools/bulk_partition_ab.py $c --reps 3 --sms 0 --no-merge-stream; done 2>&1 | cut -c1-140
echo "== C3"; timeout 900 python tools/bulk_partition_ab.py C3 --reps 1 --sms 0 | cut -c1-140
