set -x
mkdir -p gpurun_out/r2b
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r2b/smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r2b/pytest.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/r2b/pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2b/bench_c3.json 2> gpurun_out/r2b/bench_c3.err; echo "bench rc=$?"
cat gpurun_out/r2b/bench_c3.json; tail -5 gpurun_out/r2b/bench_c3.err
