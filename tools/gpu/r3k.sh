mkdir -p gpurun_out/r3k
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r3k/bench_c4.json 2> gpurun_out/r3k/bench_c4.err; echo "c4 rc=$?"
timeout 300 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3k/bench_c1.json 2> gpurun_out/r3k/bench_c1.err; echo "c1 rc=$?"
python -c "
import json
for f in ['gpurun_out/r3k/bench_c4.json','gpurun_out/r3k/bench_c1.json']:
    d=json.load(open(f)); print(f, d['config']['workload'], d['value'], d['ms_per_step'], d['roofline']['frac'], (d.get('e2e') or {}).get('value'), d['clocks'])
"
