set -x
mkdir -p gpurun_out/r2g
timeout 300 python tools/timeline.py C2 --json gpurun_out/r2g/tl_c2.json > gpurun_out/r2g/tl_c2.txt 2>&1; echo rc=$?
timeout 300 python tools/timeline.py C2 --no-lookahead --json gpurun_out/r2g/tl_c2_serial.json > gpurun_out/r2g/tl_c2_serial.txt 2>&1; echo rc=$?
timeout 300 python tools/timeline.py 8192 128 --json gpurun_out/r2g/tl_8192.json > gpurun_out/r2g/tl_8192.txt 2>&1; echo rc=$?
cat gpurun_out/r2g/tl_c2.txt gpurun_out/r2g/tl_c2_serial.txt gpurun_out/r2g/tl_8192.txt
