# late round-2 deliverables: full GPU suite (-x), smoke, bench lines c5 (default) c2 c3 c4, reference arm
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c5.log 2>&1
timeout 600 python bench.py --config c2 --steps 50 > gpurun_out/bench_c2.log 2>&1
timeout 600 python bench.py --config c3 --steps 30 > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py --config c4 --steps 20 > gpurun_out/bench_c4.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
grep -E "FAILED|passed|failed|rc=" gpurun_out/gputests.log | tail -4; tail -n 2 gpurun_out/smoke.log
for c in c5 c2 c3 c4; do tail -n 1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], '%.4g' % d['value'], '%.4f' % d['roofline']['frac'], '%.4g' % d['e2e']['value'], '%.4g' % d['train']['value'], d['train']['ms_per_step'], d['clocks'])"; done
tail -n 1 gpurun_out/bench_ref.log | cut -c1-300
