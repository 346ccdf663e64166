timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --train-steps 50 > gpurun_out/bench.log 2>&1
python tools/quickbench.py c2 22 > gpurun_out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_fwd_tc -s 10 -c 1 \
    -o gpurun_out/c2prof2 python tools/quickbench.py c2 22 > gpurun_out/ncu.log 2>&1
cat gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.log; cat gpurun_out/plain.log
