set -x
mkdir -p gpurun_out/r2q
python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/leaf_timing.py 4096 32 > gpurun_out/r2q/leaf_timing.txt 2>&1; python tools/leaf_timing.py 1024 32 >> gpurun_out/r2q/leaf_timing.txt 2>&1; grep CTA gpurun_out/r2q/leaf_timing.txt
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python tools/sanitize_run.py C1 > gpurun_out/r2q/san_racecheck_c1.log 2>&1; grep SUMMARY gpurun_out/r2q/san_racecheck_c1.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python tools/sanitize_run.py 3000 128 > gpurun_out/r2q/san_racecheck_3000.log 2>&1; grep SUMMARY gpurun_out/r2q/san_racecheck_3000.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q -k "lu or factor or degenerate or dup or kahan" > gpurun_out/r2q/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2q/pytest.log
timeout 600 python tools/schedule_ab.py C2 3 > gpurun_out/r2q/ab_c2.txt 2>&1; grep -v '^{' gpurun_out/r2q/ab_c2.txt | head -1
