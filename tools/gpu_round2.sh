# Round deliverables (all configs): GPU tests, bench lines c2..c5, the oracle arm,
# ncu launch lists of the c2 and c4 bench commands.
set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1
timeout 600 python bench.py --config c3 --cpu-sample 1048576 > gpurun_out/bench_c3.log 2>&1
timeout 600 python bench.py --config c4 --steps 20 --cpu-sample 524288 > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --config c5 --steps 10 --train-steps 20 --cpu-sample 131072 > gpurun_out/bench_c5.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 3 --warmup 3 --train-steps 3 --no-cpu-baseline > gpurun_out/ncu_launch_c2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_score_exit -c 200 --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --config c4 --steps 3 --warmup 3 --train-steps 3 --exit-train-steps 300 --no-cpu-baseline \
    > gpurun_out/ncu_launch_c4.log 2>&1
cat gpurun_out/pytest_gpu.log; for c in c2 c3 c4 c5 ref; do tail -1 gpurun_out/bench_$c.log | cut -c1-300; done
