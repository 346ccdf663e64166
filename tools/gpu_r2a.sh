# round 2, first pass: GPU tests, default bench (c5), c2 bench
set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c5.log 2>&1
timeout 600 python bench.py --config c2 --steps 50 > gpurun_out/bench_c2.log 2>&1
cat gpurun_out/pytest_gpu.log; for c in c5 c2; do tail -1 gpurun_out/bench_$c.log | cut -c1-600; done
