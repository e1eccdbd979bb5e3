mkdir -p gpurun_out/r3l
timeout 900 python tools/kahan_quality.py --sizes 1024,4096 --out gpurun_out/r3l/kahan_quality_r02b.json > gpurun_out/r3l/kahan.log 2>&1; echo "kahan rc=$?"; tail -6 gpurun_out/r3l/kahan.log
timeout 1200 python tools/run_configs.py --tols 6.03e-14,2.01e-14 --out gpurun_out/r3l/configs_r02b.json > gpurun_out/r3l/configs.log 2>&1; echo "configs rc=$?"; tail -3 gpurun_out/r3l/configs.log | cut -c1-400
