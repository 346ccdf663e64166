for d in 1 2 3; do timeout 300 python tools/hier_bench.py $d; done
