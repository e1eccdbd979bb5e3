mkdir -p gpurun_out/r3e
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3e/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r3e/smoke.log
timeout 2000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r3e/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3e/pytest.log
timeout 1200 python bench.py > gpurun_out/r3e/bench_c3.json 2> gpurun_out/r3e/bench_c3.err; echo "bench c3 rc=$?"
timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3e/bench_c2.json 2> gpurun_out/r3e/bench_c2.err; echo "bench c2 rc=$?"
python -c "
import json
for f in ['gpurun_out/r3e/bench_c3.json','gpurun_out/r3e/bench_c2.json']:
    d=json.load(open(f)); print(f, d['value'], d['ms_per_step'], d['steps'], d['warmup'], d['roofline']['frac'], d['roofline']['traffic'], (d.get('e2e') or {}).get('value'), d['clocks'], d['gpu_launches'])
"
