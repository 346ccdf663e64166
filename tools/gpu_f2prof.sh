#!/bin/bash
mkdir -p gpurun_out
for v in 2 1; do
  if [ $v = 1 ]; then export NB_FUSED1=1; fi
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 300 --csv \
    --log-file gpurun_out/f2_warm_$v.csv python tools/trainbench.py c2 20 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/f2_warm_$v.csv > gpurun_out/f2_warm_$v.txt 2>&1
  head -8 gpurun_out/f2_warm_$v.txt
done
