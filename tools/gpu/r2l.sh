set -x
mkdir -p gpurun_out/r2l
python -c "import __graft_entry__ as g; g.build()" || exit 1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py C1 > gpurun_out/r2l/san_${tool}_c1.log 2>&1; echo "$tool C1 rc=$?"; tail -3 gpurun_out/r2l/san_${tool}_c1.log
done
timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py 6000 256 > gpurun_out/r2l/san_memcheck_6000.log 2>&1; echo "memcheck 6000 rc=$?"; tail -3 gpurun_out/r2l/san_memcheck_6000.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py 12000 512 > gpurun_out/r2l/san_memcheck_12000.log 2>&1; echo "memcheck 12000 rc=$?"; tail -3 gpurun_out/r2l/san_memcheck_12000.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_run.py 3000 128 > gpurun_out/r2l/san_racecheck_3000.log 2>&1; echo "racecheck 3000 rc=$?"; tail -3 gpurun_out/r2l/san_racecheck_3000.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python -m pytest tests/test_gpu_norms.py -q -x > gpurun_out/r2l/san_memcheck_norms.log 2>&1; echo "memcheck norms rc=$?"; tail -3 gpurun_out/r2l/san_memcheck_norms.log
