mkdir -p gpurun_out/r2j
timeout 600 python -m pytest tests/test_gpu_parity.py -k "bulk_partition or lookahead_and_serial or factor_matches_oracle" -x -q > gpurun_out/r2j/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2j/pytest.log
for c in "C2" "8192 128" "16384 256"; do echo "== $c"; timeout 600 python tools/bulk_partition_ab.py $c --reps 3 --sms -1,0; done > gpurun_out/r2j/ab.txt 2>&1; cut -c1-200 gpurun_out/r2j/ab.txt
python tools/leaf_timing.py 4096 1024 lu > gpurun_out/r2j/lt.txt 2>&1; python tools/leaf_timing.py 16384 1024 lu >> gpurun_out/r2j/lt.txt 2>&1; python tools/leaf_timing.py 1024 1024 lu >> gpurun_out/r2j/lt.txt 2>&1; grep -v warning gpurun_out/r2j/lt.txt | grep "CTA\|leaf"
