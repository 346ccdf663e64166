# c2 training: per-CTA timeline of k_train_fused2 + ncu full captures of the fused kernel and the reduce
mkdir -p gpurun_out
timeout 300 python tools/trace_fused.py c2 > gpurun_out/trace_fused_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dw_reduce -s 8 -c 1 -o gpurun_out/prof_c2_reduce -f \
   timeout 300 python tools/trainbench.py c2 12 > gpurun_out/ncu_reduce.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_train_fused2 -s 8 -c 1 -o gpurun_out/prof_c2_fused2 -f \
   timeout 300 python tools/trainbench.py c2 12 > gpurun_out/ncu_fused2.log 2>&1
head -40 gpurun_out/trace_fused_c2.log; tail -n 3 gpurun_out/ncu_reduce.log gpurun_out/ncu_fused2.log
