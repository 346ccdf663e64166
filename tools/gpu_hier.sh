# hierarchy: order-preserving compaction — tests, timing, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "hier" > gpurun_out/hier_tests.log 2>&1; echo "rc=$?" >> gpurun_out/hier_tests.log
for d in 1 2 3; do timeout 300 python tools/hier_bench.py $d; done
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv --log-file gpurun_out/hier_launches.csv timeout 300 python tools/hier_bench.py 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/hier_launches.csv > gpurun_out/hier_launches.txt 2>&1
tail -n 3 gpurun_out/hier_tests.log; head -10 gpurun_out/hier_launches.txt
