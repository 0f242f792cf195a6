#!/bin/bash
# A/B builds of liblkv_b200.so with compile-time knobs, each timed by a script.
#   profiles/ab_build.sh "<script.py>" "-DKNOB=1" "-DKNOB=2" ...
set -e
cd "$(dirname "$0")/.."
script=$1; shift
for flags in "$@"; do
  tag=$(echo "$flags" | tr -c 'A-Za-z0-9' '_')
  d=/tmp/lkvab_$tag; mkdir -p $d/build
  (cd paper_2605_06676_b200 && make -s OBJDIR=$d/build LIB=$d/liblkv_b200.so NVCC="nvcc $flags" $d/liblkv_b200.so >/dev/null 2>&1)
  if [[ $script == *.sh ]]; then run="bash $script"; else run="python $script"; fi
  echo "[$flags]"; LKV_B200_LIB=$d/liblkv_b200.so $run 2>&1 | tail -4
done
