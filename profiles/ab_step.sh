#!/bin/bash
# A/B of the headline eviction step across library builds in paper_2605_06676_b200/ (alternating
# runs on the same box): profiles/ab_step.sh [reps] [lib ...] (default: in-tree vs liblkv_old.so).
# Prints ms/step, K1 ms, K3+K4 ms.
cd "$(dirname "$0")/.."
reps=${1:-3}; shift
libs=${@:-liblkv_b200.so liblkv_old.so}
for i in $(seq $reps); do
  for lib in $libs; do
    echo "$lib $(LKV_B200_LIB=$PWD/paper_2605_06676_b200/$lib python bench.py --no-e2e --no-decode --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(round(d["ms_per_step"],4), round(d["stages_ms"]["score_K1"],4), round(d["stages_ms"]["select_gather_K3K4"],4))')"
  done
done
