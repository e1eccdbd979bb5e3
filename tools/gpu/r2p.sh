mkdir -p gpurun_out/r2p
for c in "C2" "16384 256" "8192 128" "32768 512"; do echo "== $c"; timeout 900 python tools/bulk_partition_ab.py $c --reps 3 --sms -1,0,132,116,100; done > gpurun_out/r2p/ab.txt 2>&1
echo "== C3" >> gpurun_out/r2p/ab.txt; timeout 900 python tools/bulk_partition_ab.py C3 --reps 1 --sms -1,0 >> gpurun_out/r2p/ab.txt 2>&1
cut -c1-120 gpurun_out/r2p/ab.txt
