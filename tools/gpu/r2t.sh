mkdir -p gpurun_out/r2t
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2t/bench_c2.json 2> gpurun_out/r2t/bench_c2.err; echo "bench c2 rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/r2t/bench_c2.json')); print(d['value'], d['ms_per_step'], d['phase_ms_per_step']['total'], d['clocks'], (d.get('e2e') or {}).get('value'))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2t/launches_c2.csv python tools/profile_run.py C2 --warm 0 > gpurun_out/r2t/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
gzip -f gpurun_out/r2t/launches_c2.csv
