# late round-2 (session 4): new hierarchy test, c5 bench launch list + c5 score ncu capture on HEAD,
# write-only / read-only / copy HBM bandwidth (for the training kernels' store-bound roofline)
set -o pipefail
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_hierarchy.py -m gpu -x -q -p no:cacheprovider > gpurun_out/hier_tests.log 2>&1; echo "rc=$?" >> gpurun_out/hier_tests.log
python - > gpurun_out/hbm_bw.log 2>&1 <<'PY'
import torch
n = 2 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda"); b = torch.empty_like(a)
a.fill_(1); b.fill_(2); torch.cuda.synchronize()
def t(f, k=10):
    best = 1e9
    for _ in range(k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best
w = t(lambda: a.fill_(3)); print("write-only fill_ 2 GiB: %.1f GB/s" % (n / w / 1e6))
r = t(lambda: a.view(torch.int64).sum()); print("read-only sum 2 GiB: %.1f GB/s" % (n / r / 1e6))
c = t(lambda: b.copy_(a)); print("copy 2 GiB (read+write): %.1f GB/s" % (2 * n / c / 1e6))
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c5.csv \
    python bench.py --steps 3 --warmup 3 --train-steps 3 --no-cpu-baseline --model-train-steps 20 > gpurun_out/ncu_launch_c5.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c5.csv > gpurun_out/launches_c5.txt 2>&1
NB_QB_MODES=score timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fwd_tc2p -s 3 -c 1 \
    -o gpurun_out/prof_c5_score python tools/quickbench.py c5 24 > gpurun_out/ncu_c5_score.log 2>&1
ncu -i gpurun_out/prof_c5_score.ncu-rep --page raw --csv > gpurun_out/prof_c5_score_raw.csv 2>&1
tail -3 gpurun_out/hier_tests.log; cat gpurun_out/hbm_bw.log; head -8 gpurun_out/launches_c5.txt; tail -2 gpurun_out/ncu_c5_score.log
