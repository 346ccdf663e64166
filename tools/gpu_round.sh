# Round deliverables: GPU tests, bench line, ncu launch list of the bench, full ncu capture of the score kernel
set -o pipefail
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
python bench.py --steps 3 --warmup 3 --train-steps 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --train-steps 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
cat gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.log; tail -2 gpurun_out/ncu_launch.log
