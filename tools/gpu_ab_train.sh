# A/B of the c5 training step: libnb_old.so (previous build) vs libnb.so, alternating, same box
mkdir -p gpurun_out
for i in 1 2; do
  NB_LIB=old python tools/trainbench.py c5 200 >> gpurun_out/ab_train.log 2>&1
  python tools/trainbench.py c5 200 >> gpurun_out/ab_train.log 2>&1
done
cat gpurun_out/ab_train.log
