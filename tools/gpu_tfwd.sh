mkdir -p gpurun_out
for r in 1 2; do timeout 120 python tools/trainbench.py c5 100; NB_QB_MODES=score,forward timeout 200 python tools/quickbench.py c5 24; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_depth.py -x -q -p no:cacheprovider -k "c5 or pair or train or sine or pe" > gpurun_out/tfwd_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tfwd_tests.log
tail -n 2 gpurun_out/tfwd_tests.log
