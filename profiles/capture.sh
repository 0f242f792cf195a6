#!/bin/bash
# Round capture (run under gpurun, one GPU):  profiles/capture.sh r01
#  1. plain runs of every profiled command (each must exit 0 before any ncu run of it)
#  2. launch list of the bench step (cold-cache, serialised: compare shares, not absolutes)
#  3. one `ncu --set full` per hot kernel, summarised into profiles/<round>/ncu_<kernel>.txt
# Everything is written under gpurun_out/ (the only directory gpurun copies back); copy
# gpurun_out/profiles_<round>/* into profiles/<round>/ afterwards.  Optional 2nd argument: a regex of
# the kernels to capture (default: all).
set -e
R=${1:-r01}
ONLY=${2:-.}
cd "$(dirname "$0")/.."
P=gpurun_out/profiles_$R
mkdir -p $P
python profiles/step.py --evict 2 --decode 2 > gpurun_out/plain_step.log 2>&1
python profiles/attn_time.py --t 16384 --reps 2 > gpurun_out/plain_attn.log 2>&1
python profiles/model_step_time.py --eager --steps 2 > gpurun_out/plain_model.log 2>&1
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_bench_c2.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python profiles/launch_summary.py $P/launches_bench_c2.csv > $P/launches_bench_c2_summary.txt
cap() {  # kernel-regex, command...
  local k=$1; shift
  echo "$k" | grep -Eq "$ONLY" || return 0
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/${R}_$k "$@" \
      > gpurun_out/ncu_$k.log 2>&1 || true
  python profiles/summarize.py gpurun_out/${R}_$k.ncu-rep $P/ncu_$k.txt || true
}
cap score_tc python profiles/step.py --evict 2 --decode 1
cap select_plan python profiles/step.py --evict 2 --decode 1
cap select_emit python profiles/step.py --evict 2 --decode 1
cap decode_attn python profiles/step.py --evict 1 --decode 2
cap fwd_tc python profiles/attn_time.py --t 16384 --reps 1
cap dq_tc python profiles/attn_time.py --t 16384 --reps 1
cap dkv_tc python profiles/attn_time.py --t 16384 --reps 1
cap wstream_gemv python profiles/model_step_time.py --eager --steps 1
ls $P
