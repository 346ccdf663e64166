#!/bin/bash
# two-slot fused training kernel (c2): parity + timing against the one-slot kernel
mkdir -p gpurun_out
{
for c in c2; do
  echo "== $c fused2" ; timeout 120 python tools/trainbench.py $c 100
  echo "== $c fused1" ; NB_FUSED1=1 timeout 120 python tools/trainbench.py $c 100
done
} > gpurun_out/fused2_bench.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c2 or bf16_train or training or micro or adam or bit_masks or control or graph" > gpurun_out/fused2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fused2_tests.log
timeout 600 python -m pytest tests/test_gpu_depth.py -x -q -k "c2" >> gpurun_out/fused2_tests.log 2>&1; echo "depth rc=$?" >> gpurun_out/fused2_tests.log
timeout 600 python -m pytest tests/test_gpu_checked.py -x -q >> gpurun_out/fused2_tests.log 2>&1; echo "checked rc=$?" >> gpurun_out/fused2_tests.log
cat gpurun_out/fused2_bench.log
grep -E "rc=|passed|failed|Error" gpurun_out/fused2_tests.log | tail
