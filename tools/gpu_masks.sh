#!/bin/bash
# ReLU' bit masks for the single-CTA backward: parity + train-step timing
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -k "bit_masks or train or grad or sine or 4d" > gpurun_out/masks_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/masks_tests.log
python -m pytest tests/test_gpu_depth.py -x -q -k "gradient" >> gpurun_out/masks_tests.log 2>&1; echo "depth rc=$?" >> gpurun_out/masks_tests.log
for c in c2 c3 c4 c5; do
  echo "== $c masks" ; python tools/trainbench.py $c 50
  echo "== $c no masks" ; NB_NO_MASKS=1 python tools/trainbench.py $c 50
done > gpurun_out/masks_bench.log 2>&1
tail -3 gpurun_out/masks_tests.log
cat gpurun_out/masks_bench.log | grep -v "^$" | head -60
