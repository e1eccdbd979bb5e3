timeout 900 python -m pytest tests/test_gpu_parity.py -k "host or lookahead_and_serial" -x -q > gpurun_out/r3o_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r3o_pytest.log
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r3o_bench.json 2> gpurun_out/r3o_bench.err; echo "bench rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/r3o_bench.json')); print(d['value'], d['ms_per_step'], d['e2e'], d['clocks'])
"
