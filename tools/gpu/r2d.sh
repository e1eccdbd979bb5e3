set -x
mkdir -p gpurun_out/r2d
timeout 900 python tools/kahan_quality.py --sizes 1024,4096 --out gpurun_out/r2d/kahan_quality_r02.json > gpurun_out/r2d/kahan.log 2>&1; echo "kahan rc=$?"; tail -8 gpurun_out/r2d/kahan.log
timeout 600 python tools/c5_calibration.py --gpu > gpurun_out/r2d/c5cal.log 2>&1; echo "c5cal rc=$?"; cat gpurun_out/r2d/c5cal.log; cp profiles/c5_calibration_gpu_r02.json gpurun_out/r2d/ 2>/dev/null
timeout 1500 python tools/sweep.py --sizes 32768 --blocks 32,64,128,256,512,1024,2048 --variants cqr,hqr,cqr-serial,hqr-serial --reps 1 --max-iters 1100 --out gpurun_out/r2d/sweep_32768_r02.json > gpurun_out/r2d/sweep32768.log 2>&1; echo "sweep rc=$?"; tail -30 gpurun_out/r2d/sweep32768.log
timeout 1500 python tools/sweep.py --sizes 2048,4096,8192,16384 --blocks 32,64,128,256,512,1024,2048 --variants cqr,hqr --reps 2 --max-iters 600 --out gpurun_out/r2d/sweep_r02.json > gpurun_out/r2d/sweep.log 2>&1; echo "sweep rc=$?"; tail -60 gpurun_out/r2d/sweep.log
timeout 1200 python tools/run_configs.py --tols 6.03e-14,2.01e-14 --out gpurun_out/r2d/configs_r02.json > gpurun_out/r2d/configs.log 2>&1; echo "configs rc=$?"; tail -4 gpurun_out/r2d/configs.log | cut -c1-600
timeout 1800 python tools/oracle_baseline.py --c2 --out gpurun_out/r2d/oracle_baseline_r02.json > gpurun_out/r2d/oracle_baseline.log 2>&1; echo "oracle baseline rc=$?"; cat gpurun_out/r2d/oracle_baseline.log
