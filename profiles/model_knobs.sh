#!/bin/bash
# Timing-only sweep of the full decode step with launches removed (LKV_MODEL_EXPT bits: 2 attention,
# 4 qkv, 8 wo, 16 gate/up, 32 down); the deltas bound each kernel's share of the graph:
# profiles/model_knobs.sh "0 2 4 8 16 32"
cd "$(dirname "$0")/.."
for x in ${1:-0 2 4 8 16 32}; do
  echo "expt=$x $(LKV_MODEL_EXPT=$x python profiles/model_step_time.py --steps 100 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(round(d["ms_per_step"],4))')"
done
