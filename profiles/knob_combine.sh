#!/bin/bash
# Decode-step timing knobs (CUDA graph replay, Llama-3-8B geometry, C2 cache): baseline, without the
# combine kernels (LKV_NO_COMBINE, output wrong -- timing only), without the attention
# (LKV_MODEL_EXPT=2), and without the per-layer attention's early K/V prefetch (LKV_NO_EARLY_KV).
cd "$(dirname "$0")/.."
t() { python profiles/model_step_time.py --steps 100 2>/dev/null | python -c 'import json,sys; print(round(json.loads(sys.stdin.readline())["ms_per_step"],4))'; }
for i in 1 2; do
  echo "base $(t)"
  echo "no_early_kv $(LKV_NO_EARLY_KV=1 t)"
  echo "nocomb $(LKV_NO_COMBINE=1 t)"
  echo "noattn $(LKV_MODEL_EXPT=2 t)"
done
