set -o pipefail
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "train or nccl or regularized or two_shards or repack or paper_training" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_depth.py -q -x -k "gradient" 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in c2 c5; do python tools/trainbench.py $c 300; done
NB_NO_FUSED_FINALIZE=1 python tools/trainbench.py c2 300
