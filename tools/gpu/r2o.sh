set -x
mkdir -p gpurun_out/r2o
python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/leaf_timing.py 4096 32 > gpurun_out/r2o/leaf_timing.txt 2>&1; python tools/leaf_timing.py 1024 32 >> gpurun_out/r2o/leaf_timing.txt 2>&1; grep CTA gpurun_out/r2o/leaf_timing.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q -k "lu or factor or degenerate or dup or kahan" > gpurun_out/r2o/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2o/pytest.log
timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py C1 > gpurun_out/r2o/san_racecheck_c1.log 2>&1; grep SUMMARY gpurun_out/r2o/san_racecheck_c1.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py C1 > gpurun_out/r2o/san_memcheck_c1.log 2>&1; grep SUMMARY gpurun_out/r2o/san_memcheck_c1.log
timeout 600 python tools/schedule_ab.py C2 3 > gpurun_out/r2o/ab_c2.txt 2>&1; grep -v '^{' gpurun_out/r2o/ab_c2.txt | head -1
