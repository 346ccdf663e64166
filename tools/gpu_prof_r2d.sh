# training launch lists (c2, c5) + per-step times + c2 score size sweep (fixed-overhead fit)
mkdir -p gpurun_out
CONFIGS="c2 c5" bash tools/gpu_trainprof.sh > gpurun_out/trainprof.log 2>&1
for c in c2 c3 c5; do timeout 120 python tools/trainbench.py $c 100; done > gpurun_out/trainbench.log 2>&1
for k in 1 2 4 8 16 32 44; do NB_QB_MODES=score timeout 120 python tools/quickbench.py c2 22 $((740*128*k)); done > gpurun_out/c2sweep.log 2>&1
NB_QB_MODES=score timeout 120 python tools/quickbench.py c2 22 >> gpurun_out/c2sweep.log 2>&1
NB_QB_MODES=score timeout 120 python tools/quickbench.py c2 24 >> gpurun_out/c2sweep.log 2>&1
cat gpurun_out/trainprof.log gpurun_out/trainbench.log gpurun_out/c2sweep.log
