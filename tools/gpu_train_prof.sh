# steady-state training-step timing and warm-cache per-kernel durations
set -o pipefail
mkdir -p gpurun_out
for c in c2 c3 c5; do python tools/trainbench.py $c 200 >> gpurun_out/trainbench.log 2>&1; done
for c in c2 c5; do
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv \
    --log-file gpurun_out/train_warm_$c.csv python tools/trainbench.py $c 20 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/train_warm_$c.csv > gpurun_out/train_warm_$c.txt 2>&1
done
cat gpurun_out/trainbench.log; head -12 gpurun_out/train_warm_c2.txt; head -12 gpurun_out/train_warm_c5.txt
