mkdir -p gpurun_out/r2i
for c in "C2" "8192 128" "16384 256" "32768 512" "4096 64"; do echo "== $c"; timeout 600 python tools/bulk_partition_ab.py $c --reps 3 --sms -1,0,100; done > gpurun_out/r2i/ab.txt 2>&1
echo "== C3" >> gpurun_out/r2i/ab.txt; timeout 600 python tools/bulk_partition_ab.py C3 --reps 1 --sms -1,0 >> gpurun_out/r2i/ab.txt 2>&1
cat gpurun_out/r2i/ab.txt | cut -c1-330
