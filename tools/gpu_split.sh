# A/B: split D_b signal (libnb) vs single signal (libnb_nosplit)
mkdir -p gpurun_out
for r in 1 2; do
for v in "" nosplit; do
  echo "== '$v'"
  NB_LIB=$v NB_QB_MODES=score,forward timeout 200 python tools/quickbench.py c5 24
  NB_LIB=$v timeout 120 python tools/trainbench.py c5 50
done; done
