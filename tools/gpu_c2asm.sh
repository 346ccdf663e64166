set -o pipefail
timeout 120 python tools/quickbench.py c2 20 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_depth.py -q -x -k "c2 or edge or score_async or score_host or nccl or misaligned" 2>&1 | tail -3
for i in 1 2; do timeout 120 python tools/quickbench.py c2 22 2>&1 | tail -2; NB_TC_TMEM_A=1 timeout 120 python tools/quickbench.py c2 22 2>&1 | tail -2; done
