# late round-2 (session 4): hierarchy sibling-gather check + timing, c5 training warm launch list,
# one ncu --set full capture of the c5 training forward (k_fwd_tc2p kTrain)
set -o pipefail
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_hierarchy.py -m gpu -x -q -p no:cacheprovider > gpurun_out/hier_tests.log 2>&1; echo "rc=$?" >> gpurun_out/hier_tests.log
for d in 1 2 3; do timeout 300 python tools/hier_bench.py $d >> gpurun_out/hier_bench.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv \
    --log-file gpurun_out/train_warm_c5.csv python tools/trainbench.py c5 20 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/train_warm_c5.csv > gpurun_out/train_warm_c5.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fwd_tc2p" -s 5 -c 1 \
    -o gpurun_out/prof_c5train python tools/trainbench.py c5 6 > gpurun_out/ncu_c5train.log 2>&1
ncu -i gpurun_out/prof_c5train.ncu-rep --page raw --csv > gpurun_out/prof_c5train_raw.csv 2>&1
tail -3 gpurun_out/hier_tests.log; cat gpurun_out/hier_bench.log; head -14 gpurun_out/train_warm_c5.txt; tail -3 gpurun_out/ncu_c5train.log
