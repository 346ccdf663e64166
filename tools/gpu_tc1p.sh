set -o pipefail
timeout 120 python tools/quickbench.py c3 20 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_depth.py -q -x -k "c3 or plane or 4d or two_shards" 2>&1 | tail -3
for i in 1 2; do NB_QB_MODES=score,forward timeout 120 python tools/quickbench.py c3 24 2>&1 | tail -2; NB_TC1P_OFF=1 NB_QB_MODES=score,forward timeout 120 python tools/quickbench.py c3 24 2>&1 | tail -2; done
