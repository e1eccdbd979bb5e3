mkdir -p gpurun_out/r3j
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3j/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r3j/smoke.log
timeout 1200 python bench.py > gpurun_out/r3j/bench_c3.json 2> gpurun_out/r3j/bench_c3.err; echo "bench c3 rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/r3j/bench_c3.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['traffic'], (d.get('e2e') or {}).get('value'), d['clocks'], d['gpu_launches'], d['phase_ms_per_step'])
"
timeout 2000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r3j/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r3j/pytest.log
