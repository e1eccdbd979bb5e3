timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r3p_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r3p_pytest.log
