timeout 900 python -m pytest tests/test_gpu_parity.py -k "grid_leaf_cap or factor_matches or lu_pivots" -x -q > gpurun_out/r3h_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3h_pytest.log
for i in 1 2; do timeout 900 python tools/bulk_partition_ab.py C3 --reps 1 --sms 0 | cut -c1-120; done
timeout 600 python tools/bulk_partition_ab.py C2 --reps 3 --sms 0 | cut -c1-120
