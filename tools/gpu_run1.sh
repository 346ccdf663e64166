set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
for c in "c2 22" "c3 24" "c4 26" "c5 26"; do timeout 300 python tools/quickbench.py $c; done > gpurun_out/quick.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/quick.log; tail -2 gpurun_out/bench.log
