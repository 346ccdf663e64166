# full GPU suite on the spill fix, then A/B of the training steps: libnb_old.so vs libnb.so, alternating
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
for c in c5 c3 c4 c2; do for i in 1 2; do
  NB_LIB=old python tools/trainbench.py $c 200 2>&1 | sed "s/^/old /" >> gpurun_out/ab_train2.log
  python tools/trainbench.py $c 200 2>&1 | sed "s/^/new /" >> gpurun_out/ab_train2.log
done; done
grep -E "passed|failed|rc=" gpurun_out/gputests.log | tail -3; cat gpurun_out/ab_train2.log
