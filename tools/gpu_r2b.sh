# round 2: depth parity tests, recipes, compute-sanitizer
set -o pipefail
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_depth.py -q -s 2>&1 | tail -40 > gpurun_out/pytest_depth.log
timeout 1500 python tools/recipes.py --out gpurun_out/r2_recipes.json > gpurun_out/recipes.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_rc.log
done
tail -25 gpurun_out/pytest_depth.log; tail -6 gpurun_out/recipes.log | cut -c1-400; cat gpurun_out/sanitize_rc.log
for tool in memcheck racecheck synccheck; do tail -4 gpurun_out/sanitize_$tool.log; done
