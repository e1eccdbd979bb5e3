mkdir -p gpurun_out/r2k
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -k "lu or factor_matches or degenerate or duplicate or c1_seeds or bench_block" -x -q > gpurun_out/r2k/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2k/pytest.log
for c in "C2" "8192 128"; do echo "== $c"; timeout 600 python tools/bulk_partition_ab.py $c --reps 3 --sms 0; done > gpurun_out/r2k/ab.txt 2>&1; cut -c1-250 gpurun_out/r2k/ab.txt
(python tools/leaf_timing.py 4096 1024 lu; python tools/leaf_timing.py 16384 1024 lu; python tools/leaf_timing.py 1024 32 qr; python tools/leaf_timing.py 2048 32 qr) > gpurun_out/r2k/lt.txt 2>&1; grep -v warning gpurun_out/r2k/lt.txt | grep "CTA\|leaf"
