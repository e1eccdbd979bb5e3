set -x
python tools/leaf_timing.py 4096 32 > gpurun_out/r2n/leaf_timing.txt 2>&1; python tools/leaf_timing.py 1024 32 >> gpurun_out/r2n/leaf_timing.txt 2>&1; cat gpurun_out/r2n/leaf_timing.txt
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r2n/bench_c3.json 2> gpurun_out/r2n/bench_c3.err; echo "bench rc=$?"; cat gpurun_out/r2n/bench_c3.json; tail -3 gpurun_out/r2n/bench_c3.err
timeout 900 ncu --set full --clock-control none -k regex:"gather_cols_kernel|scatter_cols_kernel|col_norms_kernel|trailing_rows_kernel" -c 8 -o gpurun_out/r2n/hbm_kernels python tools/hbm_probe.py > gpurun_out/r2n/ncu_hbm.log 2>&1; echo "ncu hbm rc=$?"; tail -3 gpurun_out/r2n/ncu_hbm.log
