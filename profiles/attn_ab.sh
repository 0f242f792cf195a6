#!/bin/bash
# A/B builds of the attention kernels with LKV_ATTN_EXPT bisection knobs (run on the GPU box):
#   profiles/attn_ab.sh "0 1 2 3"   -> one library per knob value, timing of each
set -e
cd "$(dirname "$0")/.."
for x in ${1:-0 1 2 3}; do
  make -s -C paper_2605_06676_b200 OBJDIR=build_ab$x LIB=liblkv_ab$x.so NVCC="nvcc -DLKV_ATTN_EXPT=$x" liblkv_ab$x.so >/dev/null
  echo "EXPT=$x $(LKV_B200_LIB=$PWD/paper_2605_06676_b200/liblkv_ab$x.so python profiles/attn_time.py --t 8192 --nocheck 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("fwd_ms", round(d["fwd_ms"],3), "bwd_ms", round(d["bwd_ms"],3))')"
done
