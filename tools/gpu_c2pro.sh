# c2 score after overlapping the first record loads with the weight load
mkdir -p gpurun_out
for r in 1 2 3; do NB_QB_MODES=score timeout 120 python tools/quickbench.py c2 22; done
for k in 1 2; do NB_QB_MODES=score timeout 120 python tools/quickbench.py c2 22 $((740*128*k)); done
NB_QB_MODES=score timeout 200 python tools/quickbench.py c3 24
timeout 600 python bench.py --config c2 --steps 50 > gpurun_out/bench_c2.log 2>&1
tail -n 1 gpurun_out/bench_c2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_ms_per_launch'], d['clocks'])"
