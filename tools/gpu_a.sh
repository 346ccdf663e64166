timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
for c in c2 c3 c4 c5; do timeout 300 python tools/trainbench.py $c 30; done > gpurun_out/train.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/train.log
