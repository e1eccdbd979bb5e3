set -x
mkdir -p gpurun_out/r2p
python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/leaf_timing.py 4096 32 > gpurun_out/r2p/leaf_timing.txt 2>&1; grep CTA gpurun_out/r2p/leaf_timing.txt
for r in 1024 2048 4096; do python tools/leaf_probe.py qr $r 5; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q > gpurun_out/r2p/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2p/pytest.log
for t in racecheck memcheck synccheck; do timeout 600 compute-sanitizer --tool $t --print-limit 10 python tools/sanitize_run.py C1 > gpurun_out/r2p/san_${t}_c1.log 2>&1; grep SUMMARY gpurun_out/r2p/san_${t}_c1.log; done
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python tools/sanitize_run.py 3000 128 > gpurun_out/r2p/san_racecheck_3000.log 2>&1; grep SUMMARY gpurun_out/r2p/san_racecheck_3000.log
timeout 600 python tools/schedule_ab.py C2 3 > gpurun_out/r2p/ab_c2.txt 2>&1; grep -v '^{' gpurun_out/r2p/ab_c2.txt | head -1
