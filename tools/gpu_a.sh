timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
for st in 2 3 4; do echo "stages $st"; NB_DW_STAGES=$st timeout 300 python tools/trainbench.py c2 50; NB_DW_STAGES=$st timeout 300 python tools/trainbench.py c4 50; done > gpurun_out/train.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/train.log
