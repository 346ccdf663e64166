# final c5: bench launch list (the same command as the driver's, short) + ncu full capture of the score kernel
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --train-steps 3 --no-cpu-baseline --model-train-steps 20 > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c5.csv \
    python bench.py --steps 3 --warmup 3 --train-steps 3 --no-cpu-baseline --model-train-steps 20 > gpurun_out/ncu_launch_c5.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c5.csv > gpurun_out/launches_c5.txt 2>&1
NB_QB_MODES=score ncu --set full --clock-control none --import-source on -k regex:k_fwd_tc2p -s 3 -c 1 \
    -o gpurun_out/prof_c5_score -f python tools/quickbench.py c5 24 > gpurun_out/ncu_c5_score.log 2>&1
head -12 gpurun_out/launches_c5.txt; tail -n 2 gpurun_out/ncu_c5_score.log
