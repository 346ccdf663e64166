set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c5.log 2>&1
cat gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench_c5.log | cut -c1-300
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_c5.log').read().strip().splitlines()[-1])
print(d['value'], d['roofline'], d['e2e'], d['clocks'], d.get('train'))
PY
