# session 5 A/B: NB_EXP (early record staging by thread 0, weight wait deferred to the MMA warp) on c2
mkdir -p gpurun_out
timeout 300 python tools/sanitize.py fwd_c2 > gpurun_out/san_base.json 2>gpurun_out/san_base.err
timeout 300 python tools/sanitize.py --lib exp fwd_c2 > gpurun_out/san_exp.json 2>gpurun_out/san_exp.err
cmp gpurun_out/san_base.json gpurun_out/san_exp.json && echo "DIGESTS EQUAL" || { echo "DIGESTS DIFFER"; tail -3 gpurun_out/san_exp.err; }
for i in 1 2 3 4; do
  echo "base:"; timeout 120 python tools/quickbench.py c2 22 2>&1 | tail -2
  echo "exp:";  NB_LIB=exp timeout 120 python tools/quickbench.py c2 22 2>&1 | tail -2
done
