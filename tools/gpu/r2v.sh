mkdir -p gpurun_out/r2v
timeout 900 python -m pytest tests/test_gpu_parity.py -k "early_a5 or factor_matches or pipelined or lookahead_and_serial or kahan or graded or breakdown" -x -q > gpurun_out/r2v/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2v/pytest.log | grep -v "^  "
for c in "C2" "8192 128" "16384 256" "4096 64" "32768 512"; do echo "== $c"; timeout 600 python tools/bulk_partition_ab.py $c --reps 3 --sms 0; timeout 600 python tools/bulk_partition_ab.py $c --reps 3 --sms 0 --no-early; done 2>&1 | cut -c1-330
echo "== C3"; timeout 900 python tools/bulk_partition_ab.py C3 --reps 1 --sms 0 | cut -c1-330
