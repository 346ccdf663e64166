#!/bin/bash
# per-segment durations of the early-exit score kernels (dev tool; GPU box)
# usage: tools/exit_ncu.sh [NB_LIB variant ...]
for v in "" "$@"; do
  echo "== variant '${v:-main}'"
  NB_LIB=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_score_exit -c 3 \
    python tools/exit_bench.py 3000 26 2>&1 | grep -E "k_score_exit<|duration|compact|dense" | sed -e 's/(unnamed>::ExitParams).*//'
done
