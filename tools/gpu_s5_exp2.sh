# session 5 A/B: NB_EXP2 (score-mode counts in per-lane registers, one warp reduction after the tile loop) on c2
mkdir -p gpurun_out
timeout 300 python tools/sanitize.py fwd_c2 > gpurun_out/san_base.json 2>gpurun_out/san_base.err
timeout 300 python tools/sanitize.py --lib exp2 fwd_c2 > gpurun_out/san_exp2.json 2>gpurun_out/san_exp2.err
cmp gpurun_out/san_base.json gpurun_out/san_exp2.json && echo "DIGESTS EQUAL" || { echo "DIGESTS DIFFER"; cat gpurun_out/san_base.json gpurun_out/san_exp2.json; tail -3 gpurun_out/san_exp2.err; }
for i in 1 2 3 4; do
  echo "base:"; NB_QB_MODES=score timeout 120 python tools/quickbench.py c2 22 2>&1 | tail -1
  echo "exp2:"; NB_QB_MODES=score NB_LIB=exp2 timeout 120 python tools/quickbench.py c2 22 2>&1 | tail -1
done
