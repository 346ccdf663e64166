for i in 1 2 3; do timeout 300 python tools/quickbench.py c2 22; NB_LIB=split timeout 300 python tools/quickbench.py c2 22; done > gpurun_out/quick.log 2>&1
NB_LIB=split timeout 600 python -m pytest tests -m gpu -x -q -k "c2" 2>&1 | tail -2 >> gpurun_out/quick.log
cat gpurun_out/quick.log
