# pair-kernel timeline (CTA 0)
mkdir -p gpurun_out
timeout 300 python tools/trace_tc2.py 20 > gpurun_out/trace_tc2.log 2>&1
cat gpurun_out/trace_tc2.log | tail -n 24; head -n 80 gpurun_out/trace_tc2.log | tail -n 40
