# usage: bash tools/gpu_prof.sh <cfg> <logn> <launch-skip> <tag>
cfg=$1; logn=$2; skip=$3; tag=$4
python tools/quickbench.py $cfg $logn > gpurun_out/plain_$tag.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_fwd_tc -s $skip -c 1 \
    -o gpurun_out/prof_$tag python tools/quickbench.py $cfg $logn > gpurun_out/ncu_$tag.log 2>&1
tail -3 gpurun_out/ncu_$tag.log
