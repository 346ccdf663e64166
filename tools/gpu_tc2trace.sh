# pair-kernel timeline (CTA 0) + c5 pair-kernel tests + c5 quick timing
mkdir -p gpurun_out
timeout 300 python tools/trace_tc2.py 20 > gpurun_out/trace_tc2.log 2>&1
NB_QB_MODES=score timeout 200 python tools/quickbench.py c5 24 > gpurun_out/qb_c5.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_depth.py tests/test_gpu_checked.py -x -q -p no:cacheprovider -k "c5 or pair or checked or release" > gpurun_out/tc2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc2_tests.log
tail -n 25 gpurun_out/trace_tc2.log; cat gpurun_out/qb_c5.log; tail -n 2 gpurun_out/tc2_tests.log
