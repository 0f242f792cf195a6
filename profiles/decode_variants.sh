#!/bin/bash
# A/B builds of the decode kernel (stages x CTAs/SM) timed on the C2 decode loop.
set -e
cd "$(dirname "$0")/.."
for v in "3 2" "4 1" "4 2" "2 2"; do
  set -- $v
  d=/tmp/lkvvar_$1_$2; mkdir -p $d/build
  (cd paper_2605_06676_b200 && make -s OBJDIR=$d/build LIB=$d/liblkv_b200.so NVCC="nvcc -DLKV_DEC_STAGES=$1 -DLKV_DEC_PER_SM=$2" >/dev/null)
  echo "stages=$1 per_sm=$2: $(LKV_B200_LIB=$d/liblkv_b200.so python profiles/decode_time.py)"
done
