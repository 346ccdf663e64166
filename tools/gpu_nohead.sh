mkdir -p gpurun_out
for v in "" nohead; do
ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max --clock-control none --cache-control none -c 250 --csv \
    --log-file gpurun_out/rh_$v.csv timeout 120 env NB_LIB=$v python tools/trainbench.py c2 6 > /dev/null 2>&1
echo "== '$v'"; grep -E "k_dw_reduce" gpurun_out/rh_$v.csv | tail -3 | awk -F'","' '{print $(NF-3), $(NF-1), $NF}'
NB_LIB=$v timeout 120 python tools/trainbench.py c2 200
done
