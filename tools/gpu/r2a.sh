set -x
nproc; lscpu | grep "Model name"
mkdir -p gpurun_out/r2a
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -k "not factor_c2 and not factor_bench and not b4096" -x -q > gpurun_out/r2a/pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2a/pytest.log
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py C1 > gpurun_out/r2a/san_${tool}_c1.log 2>&1; echo "$tool C1 rc=$?"; tail -3 gpurun_out/r2a/san_${tool}_c1.log
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py 8192 1024 > gpurun_out/r2a/san_memcheck_8192.log 2>&1; echo "memcheck 8192 rc=$?"; tail -3 gpurun_out/r2a/san_memcheck_8192.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_run.py 8192 1024 > gpurun_out/r2a/san_racecheck_8192.log 2>&1; echo "racecheck 8192 rc=$?"; tail -3 gpurun_out/r2a/san_racecheck_8192.log
