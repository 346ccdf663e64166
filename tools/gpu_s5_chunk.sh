# session 5: early-exit compaction chunk-size sweep on the c4 bench (env knob, no rebuild)
mkdir -p gpurun_out
for lg in 22 23 24 25 26; do
  NB_EXIT_CHUNK=$((1<<lg)) timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --train-steps 3 > gpurun_out/c4_chunk_$lg.log 2>&1
  tail -n 1 gpurun_out/c4_chunk_$lg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunk 2^$lg', '%.4g q/s' % d['value'], '%.3f ms' % d['ms_per_step'], 'frac %.4f' % d['roofline']['frac'], 'dense %.3f ms' % d['early_exit']['dense_kernel_ms_per_step'])"
done | tee gpurun_out/c4_chunk_sweep.txt
