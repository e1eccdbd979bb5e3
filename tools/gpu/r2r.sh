set -x
mkdir -p gpurun_out/r2r
python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/leaf_timing.py 4096 32 lu > gpurun_out/r2r/leaf_timing.txt 2>&1; python tools/leaf_timing.py 2048 32 qr >> gpurun_out/r2r/leaf_timing.txt 2>&1; python tools/leaf_timing.py 1024 32 qr >> gpurun_out/r2r/leaf_timing.txt 2>&1; grep CTA gpurun_out/r2r/leaf_timing.txt
timeout 600 python tools/schedule_ab.py C2 3 > gpurun_out/r2r/ab_c2.txt 2>&1; grep -v '^{' gpurun_out/r2r/ab_c2.txt | head -1
