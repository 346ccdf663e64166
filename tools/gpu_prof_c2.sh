# ncu full capture of the c2 score kernel (one launch) + MMA microbenchmarks
./tools/tmem_bench > gpurun_out/tmem_bench.log 2>&1
python tools/quickbench.py c2 22 > gpurun_out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_fwd_tc -s 10 -c 1 \
    -o gpurun_out/c2prof python tools/quickbench.py c2 22 > gpurun_out/ncu.log 2>&1
tail -5 gpurun_out/ncu.log
