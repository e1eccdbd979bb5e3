mkdir -p gpurun_out/r2x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2x/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2x/smoke.log
timeout 2000 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/r2x/pytest.log 2>&1; echo "pytest rc=$?"; tail -22 gpurun_out/r2x/pytest.log
