mkdir -p gpurun_out/r2w
timeout 1200 python -m pytest tests/test_gpu_parity.py -k "early_a5 or factor_matches or pipelined or lookahead_and_serial or kahan or graded or breakdown" -v --timeout=150 -p no:cacheprovider > gpurun_out/r2w/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "PASSED|FAILED|ERROR|Timeout" gpurun_out/r2w/pytest.log | cut -c1-150 | head -60
