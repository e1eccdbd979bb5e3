set -x
mkdir -p gpurun_out/r2k
python -c "import __graft_entry__ as g; g.build()" || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/dsmem_bench tools/dsmem_bench.cu && /tmp/dsmem_bench > gpurun_out/r2k/dsmem_bench.txt 2>&1; cat gpurun_out/r2k/dsmem_bench.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q -k "sketch_qr or factor or panel or hqr or householder or kahan or lookahead" > gpurun_out/r2k/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2k/pytest.log
python tools/leaf_probe.py qr 2048 5 > gpurun_out/r2k/leaf_probe.txt 2>&1; cat gpurun_out/r2k/leaf_probe.txt
timeout 600 python tools/schedule_ab.py C2 3 > gpurun_out/r2k/ab_c2.txt 2>&1; grep -v '^{' gpurun_out/r2k/ab_c2.txt | head -1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:qr_leaf_fast -s 2 -c 1 -o gpurun_out/r2k/qr_fast_2048 python tools/leaf_probe.py qr 2048 2 > gpurun_out/r2k/ncu_qr.log 2>&1; echo "ncu qr rc=$?"
