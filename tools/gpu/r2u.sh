mkdir -p gpurun_out/r2u
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/r2u/bench_c3.json 2> gpurun_out/r2u/bench_c3.err; echo "bench c3 rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/r2u/bench_c3.json')); print(d['value'], d['ms_per_step'], d['phase_ms_per_step']['total'], d['roofline']['frac'], d['clocks'], (d.get('e2e') or {}).get('value'))"
timeout 3000 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2u/launches_c3.csv python tools/profile_run.py C3 --warm 0 > gpurun_out/r2u/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
gzip -f gpurun_out/r2u/launches_c3.csv
