set -x
mkdir -p gpurun_out/r2f
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f/launches_c2.csv python tools/profile_run.py C2 --warm 0 > gpurun_out/r2f/ncu_c2.log 2>&1; echo "ncu list rc=$?"
timeout 300 python tools/profile_run.py C2 --no-lookahead > gpurun_out/r2f/c2_serial.txt 2>&1; echo "serial rc=$?"; tail -5 gpurun_out/r2f/c2_serial.txt
for r in 1024 2048 4096 8192 16384 32768 63488; do python tools/leaf_probe.py lu $r 5; done > gpurun_out/r2f/leaf_lu.txt 2>&1; cat gpurun_out/r2f/leaf_lu.txt
for r in 1024 2048; do python tools/leaf_probe.py qr $r 5; done > gpurun_out/r2f/leaf_qr.txt 2>&1; cat gpurun_out/r2f/leaf_qr.txt
gzip -f gpurun_out/r2f/launches_c2.csv
