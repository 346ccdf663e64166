timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/bench.log 2>&1
cat gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['train'])"
