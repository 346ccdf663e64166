# round-2 session 5: bench lines c2 c3 c4 and the reference arm re-measured on HEAD
mkdir -p gpurun_out
timeout 600 python bench.py --config c2 --steps 50 > gpurun_out/bench_c2.log 2>&1
timeout 600 python bench.py --config c3 --steps 30 > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py --config c4 --steps 20 > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
for c in c2 c3 c4; do tail -n 1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], '%.4g' % d['value'], '%.4f' % d['roofline']['frac'], '%.4g' % d['e2e']['value'], '%.4g' % d['train']['value'], d['train']['ms_per_step'], d['clocks'])"; done
tail -n 1 gpurun_out/bench_ref.log | cut -c1-300
