mkdir -p gpurun_out/r2r2
(timeout 600 python tools/bulk_partition_ab.py C2 --reps 4 --sms 0,-1; timeout 600 python tools/bulk_partition_ab.py C2 --reps 4 --sms 0,-1 --phases) 2>&1 | cut -c1-100
./tools/green_probe 132 2>&1 | tail -8
