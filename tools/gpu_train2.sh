set -o pipefail
for c in c2 c5; do python tools/trainbench.py $c 200; done
NB_TC2_SINGLE=1 python tools/quickbench.py c5 24 | tail -2
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "c5" 2>&1 | tail -2
