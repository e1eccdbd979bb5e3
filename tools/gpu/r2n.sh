mkdir -p gpurun_out/r2n
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2n/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2n/pytest.log
