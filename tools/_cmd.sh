python tools/e2e_breakdown.py
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py tests/test_gpu_golden.py tests/test_controlled.py -x -q 2>&1 | tail -2
python bench.py --no-policy --no-cpu-baseline > gpurun_out/bench_e2e.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/bench_e2e.json').read().splitlines()[-1]); print(d['value'], d['e2e'])"
