timeout 600 python bench.py --steps 20 --train-steps 20 > gpurun_out/bench_c2.log 2>&1
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --steps 5 --train-steps 10 --cpu-sample 65536 > gpurun_out/bench_$c.log 2>&1; done
for c in c2 c3 c4 c5; do tail -1 gpurun_out/bench_$c.log | cut -c1-400; done
