#!/bin/bash
# A/B of the headline eviction step between the in-tree library and paper_2605_06676_b200/liblkv_old.so
# on the same box (alternating runs): profiles/ab_step.sh [reps]
cd "$(dirname "$0")/.."
for i in $(seq ${1:-3}); do
  for lib in liblkv_b200.so liblkv_old.so; do
    echo "$lib $(LKV_B200_LIB=$PWD/paper_2605_06676_b200/$lib python bench.py --no-e2e --no-decode --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(round(d["ms_per_step"],4), round(d["stages_ms"]["score_K1"],4), round(d["stages_ms"]["select_gather_K3K4"],4))')"
  done
done
