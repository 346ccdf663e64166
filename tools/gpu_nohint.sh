# mbarrier suspend-hint A/B: c5 scoring and training
mkdir -p gpurun_out
for v in "" nohint "" nohint; do
  echo "== variant '${v}'"
  NB_LIB=$v timeout 120 python tools/trainbench.py c5 50
  NB_LIB=$v NB_QB_MODES=score timeout 200 python tools/quickbench.py c5 24
done
