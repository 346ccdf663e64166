timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 300 python tools/quickbench.py c5 24; done > gpurun_out/quick.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/quick.log
