mkdir -p gpurun_out
for r in 1 2; do timeout 120 python tools/trainbench.py c2 200; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_depth.py -x -q -p no:cacheprovider -k "c2 or train or grad or adam or micro or graph or control or two_shards" > gpurun_out/headT_tests.log 2>&1; echo "rc=$?" >> gpurun_out/headT_tests.log
tail -n 3 gpurun_out/headT_tests.log
