mkdir -p gpurun_out/r2y
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py C1 > gpurun_out/r2y/san_${tool}_c1_r02b.log 2>&1; echo "$tool C1 rc=$?"; tail -2 gpurun_out/r2y/san_${tool}_c1_r02b.log
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_run.py 4096 512 --lula > gpurun_out/r2y/san_memcheck_4096_lula_r02b.log 2>&1; echo "memcheck 4096 lula rc=$?"; tail -2 gpurun_out/r2y/san_memcheck_4096_lula_r02b.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_run.py 4096 512 > gpurun_out/r2y/san_racecheck_4096_r02b.log 2>&1; echo "racecheck 4096 rc=$?"; tail -2 gpurun_out/r2y/san_racecheck_4096_r02b.log
timeout 1500 python tools/sweep.py --sizes 2048,4096,8192,16384 --blocks 64,128,256,512,1024,2048 --variants cqr --reps 2 --max-iters 600 --out gpurun_out/r2y/sweep_r02b.json > gpurun_out/r2y/sweep.log 2>&1; echo "sweep rc=$?"; tail -30 gpurun_out/r2y/sweep.log | cut -c1-160
