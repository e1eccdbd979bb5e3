for L in 16 24 32 48 0 32; do timeout 900 python tools/bulk_partition_ab.py C3 --reps 1 --sms 0 --lu-grid $L | cut -c1-200 | sed "s/^/lu_grid=$L /"; done
