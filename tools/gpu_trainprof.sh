#!/bin/bash
# warm per-kernel durations of training steps (ncu launch list)
mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c3 c5}; do
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 200 --csv \
    --log-file gpurun_out/tp_$c.csv timeout 120 python tools/trainbench.py $c 12 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/tp_$c.csv > gpurun_out/tp_$c.txt 2>&1
  echo "== $c"; head -9 gpurun_out/tp_$c.txt | tail -7
done
