# session 5: warm ncu launch lists of the c2 / c3 / c4 training steps on HEAD and one full
# capture of the fused c2 training kernel (tensor pipe, DRAM bytes, issue activity)
mkdir -p gpurun_out
CONFIGS="c2 c3 c4" bash tools/gpu_trainprof.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_train_fused -s 6 -c 1 \
    -o gpurun_out/prof_c2_train python tools/trainbench.py c2 12 > gpurun_out/ncu_c2_train.log 2>&1
ncu -i gpurun_out/prof_c2_train.ncu-rep --page raw --csv > gpurun_out/prof_c2_train_raw.csv 2>&1
python - <<'PY'
import csv
r = list(csv.reader(open('gpurun_out/prof_c2_train_raw.csv')))
h, u, v = r[0], r[1], r[2]
for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
          "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
          "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
          "sm__warps_active.avg.pct_of_peak_sustained_active"):
    if k in h:
        i = h.index(k); print(k, "=", v[i], u[i])
PY
