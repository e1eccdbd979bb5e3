for L in 0 64 32; do timeout 900 python tools/bulk_partition_ab.py C3 --reps 1 --sms 0 --lu-grid $L | cut -c1-330; done
