# per-segment durations and DRAM bytes: record vs image hand-off (c4, 2^26, model trained 2000 steps)
mkdir -p gpurun_out
for v in rec img; do
  if [ $v = img ]; then export NB_EXIT_IMAGES=1; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_score_exit -c 6 \
    python tools/exit_bench.py 2000 26 > gpurun_out/exitncu_$v.log 2>&1
  echo "== $v"; grep -E "k_score_exit|duration|dram__|tensor" gpurun_out/exitncu_$v.log | sed -e 's/(nb::.*ExitParams).*//' | head -30
done
