set -o pipefail
mkdir -p gpurun_out
timeout 120 python tools/quickbench.py c5 20 > gpurun_out/qb_c5_small.log 2>&1; echo "small rc=$?"
tail -2 gpurun_out/qb_c5_small.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "c5 or edge or two_shards" 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_depth.py -q -x -k "c5" 2>&1 | tail -2
timeout 120 python tools/quickbench.py c5 24 2>&1 | tail -2
python tools/trace_tc2.py 20 --rebuild > gpurun_out/trace_tc2.log 2>&1; tail -22 gpurun_out/trace_tc2.log
