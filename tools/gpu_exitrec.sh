# c4 early exits: both hand-offs in the tests; c4 bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "exit" > gpurun_out/exitrec_tests.log 2>&1; echo "rc=$?" >> gpurun_out/exitrec_tests.log
timeout 900 python bench.py --config c4 --steps 20 > gpurun_out/bench_c4.log 2>&1
tail -n 3 gpurun_out/exitrec_tests.log; tail -n 1 gpurun_out/bench_c4.log | cut -c1-3000
