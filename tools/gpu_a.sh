timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
for c in c2; do timeout 300 python tools/trainbench.py $c 50; NB_NO_FUSED=1 timeout 300 python tools/trainbench.py $c 50; done > gpurun_out/train.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/train.log
