# ncu full capture of the c5 training forward (k_fwd_tc2p kTrain)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_fwd_tc2p -s 3 -c 1 -o gpurun_out/prof_c5_trainfwd -f \
   timeout 300 python tools/trainbench.py c5 8 > gpurun_out/ncu_trainfwd.log 2>&1
tail -n 2 gpurun_out/ncu_trainfwd.log
