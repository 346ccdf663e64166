#!/bin/bash
for c in c2 c3 c5; do
  echo "== $c fused adam"; timeout 60 python tools/trainbench.py $c 100
  echo "== $c separate"; NB_ADAM_SEPARATE=1 timeout 60 python tools/trainbench.py $c 100
done
CONFIGS="c2 c5" ./tools/gpu_trainprof.sh
export NB_ADAM_SEPARATE=1; CONFIGS="c2 c5" ./tools/gpu_trainprof.sh
