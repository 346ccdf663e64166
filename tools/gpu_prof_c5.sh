# c5 score kernel: one ncu --set full capture; NCCL launch list of the world-1 communicator test
set -o pipefail
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_fwd_tc2p -s 6 -c 1 \
    -o gpurun_out/prof_c5p python tools/quickbench.py c5 24 > gpurun_out/ncu_c5p.log 2>&1
tail -2 gpurun_out/ncu_c5p.log
ncu -i gpurun_out/prof_c5p.ncu-rep --page raw --csv > gpurun_out/prof_c5p_raw.csv 2>&1
python tools/ncu_to_summary.py gpurun_out/prof_c5p.ncu-rep c5 "k_fwd_tc2p<4,kScore,d0=6> (pipelined CTA pairs)" \
  "ncu --set full --clock-control none, 1 launch of the c5 kernel at n = 2^24 (tools/quickbench.py c5 24, launch 7); the bench step is 2^28 rows = 16x this launch's bytes" | head -30
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_nccl.csv \
    python -m pytest tests/test_gpu_parity.py -q -k nccl > gpurun_out/ncu_nccl.log 2>&1
tail -2 gpurun_out/ncu_nccl.log
python tools/launch_summary.py gpurun_out/launches_nccl.csv > gpurun_out/launches_nccl.txt; grep -i nccl gpurun_out/launches_nccl.txt
