mkdir -p gpurun_out/r2q
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r2q/bench_c3.json 2> gpurun_out/r2q/bench_c3.err; echo "bench c3 rc=$?"
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2q/bench_c2.json 2> gpurun_out/r2q/bench_c2.err; echo "bench c2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2q/launches_c2.csv python tools/profile_run.py C2 --warm 0 > gpurun_out/r2q/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2q/launches_c3.csv python tools/profile_run.py C3 --warm 0 > gpurun_out/r2q/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
gzip -f gpurun_out/r2q/launches_c2.csv gpurun_out/r2q/launches_c3.csv
python -c "
import json
for f in ['gpurun_out/r2q/bench_c3.json','gpurun_out/r2q/bench_c2.json']:
    d=json.load(open(f)); print(f, d['value'], d['ms_per_step'], d['roofline']['frac'], (d.get('e2e') or {}).get('value'), d['clocks'])
"
