mkdir -p gpurun_out/r3d
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dgemm2 -c 1 -o gpurun_out/r3d/ncu_full_bulk_gemm2_g32_c3_r02 ./tools/gsp_g32 > gpurun_out/r3d/ncu_full.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/r3d/ncu_full_bulk_gemm2_g32_c3_r02.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2] if len(rows)>2 else rows[1]
want=['dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fp64.sum','lts__t_sector_hit_rate.pct']
for w in want:
    for i,x in enumerate(h):
        if x==w: print(w, rows[1][i], v[i])
"
for c in "C2" "8192 256"; do timeout 600 python tools/bulk_partition_ab.py $c --reps 3 --sms 0 | cut -c1-110; done
for i in 1 2; do timeout 900 python tools/bulk_partition_ab.py C3 --reps 1 --sms 0 | cut -c1-110; done
