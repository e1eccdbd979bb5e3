set -x
mkdir -p gpurun_out/r2g
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g/launches_c2.csv python tools/profile_run.py C2 > gpurun_out/r2g/ncu_c2.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:qr_leaf_fast -s 2 -c 1 -o gpurun_out/r2g/qr_fast_2048 python tools/leaf_probe.py qr 2048 2 > gpurun_out/r2g/ncu_qr.log 2>&1; echo "ncu qr rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:trsm_base -s 20 -c 3 -o gpurun_out/r2g/trsm_base python tools/profile_run.py C2 --warm 0 > gpurun_out/r2g/ncu_trsm.log 2>&1; echo "ncu trsm rc=$?"
