set -o pipefail
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c5 and (train or regularized or repack or two_shards)" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_depth.py -q -x -k "gradient and c5" 2>&1 | tail -2
python tools/trainbench.py c5 300
NB_TC2_SINGLE=1 python tools/trainbench.py c5 300
