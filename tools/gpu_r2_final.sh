# round-2 deliverables: bench lines c2..c5, reference arm, c5 launch list, c5 score ncu capture
set -o pipefail
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c5.log 2>&1
timeout 600 python bench.py --config c2 --steps 50 > gpurun_out/bench_c2.log 2>&1
timeout 600 python bench.py --config c3 --steps 30 > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py --config c4 --steps 20 > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
python bench.py --steps 3 --warmup 3 --train-steps 3 --no-cpu-baseline --model-train-steps 20 > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c5.csv \
    python bench.py --steps 3 --warmup 3 --train-steps 3 --no-cpu-baseline --model-train-steps 20 > gpurun_out/ncu_launch_c5.log 2>&1
NB_QB_MODES=score ncu --set full --clock-control none --import-source on -k regex:k_fwd_tc2p -s 3 -c 1 \
    -o gpurun_out/prof_c5_score python tools/quickbench.py c5 24 > gpurun_out/ncu_c5_score.log 2>&1
for c in c5 c2 c3 c4 ref; do tail -1 gpurun_out/bench_$c.log | cut -c1-200; done
tail -2 gpurun_out/ncu_c5_score.log
