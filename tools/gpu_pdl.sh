# PDL variants for the fused c2 step
mkdir -p gpurun_out
for rep in 1 2; do
echo "== both"; timeout 120 python tools/trainbench.py c2 300
echo "== no fused pdl"; NB_NO_PDL_FUSED=1 timeout 120 python tools/trainbench.py c2 300
echo "== no reduce pdl"; NB_NO_PDL_REDUCE=1 timeout 120 python tools/trainbench.py c2 300
echo "== none"; NB_NO_PDL_FUSED=1 NB_NO_PDL_REDUCE=1 timeout 120 python tools/trainbench.py c2 300
done
