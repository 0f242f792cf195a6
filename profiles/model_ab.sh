#!/bin/bash
# A/B of the full decode step (model_step_time.py) across library builds in paper_2605_06676_b200/,
# alternating runs on the same box: profiles/model_ab.sh [reps] [lib ...] (default: in-tree vs liblkv_old.so)
cd "$(dirname "$0")/.."
reps=${1:-2}; shift
libs=${@:-liblkv_b200.so liblkv_old.so}
for i in $(seq $reps); do
  for lib in $libs; do
    echo "$lib $(LKV_B200_LIB=$PWD/paper_2605_06676_b200/$lib python profiles/model_step_time.py --steps 100 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(round(d["ms_per_step"],4), round(d["frac_of_measured_hbm"],3))')"
  done
done
