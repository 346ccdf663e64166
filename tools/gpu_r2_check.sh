# round-2 check: full GPU suite (-x as the driver runs it), smoke
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
grep -E "FAILED|passed|failed|rc=" gpurun_out/gputests.log | tail; tail -n 2 gpurun_out/smoke.log
