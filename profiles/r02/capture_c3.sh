#!/bin/bash
# Round-2 capture on the C3 headline (run under gpurun, one GPU): launch list of the bench command
# and one `ncu --set full` per hot kernel, summaries into gpurun_out/profiles_r02/.
cd "$(dirname "$0")/../.."
P=gpurun_out/profiles_r02
mkdir -p $P
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-sweep"
S="python profiles/step.py --config 3 --evict 2 --decode 2"
$B > gpurun_out/plain_bench.log 2>&1 || exit 1
$S > gpurun_out/plain_step.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_bench_c3.csv $B > /dev/null 2>&1
python profiles/launch_summary.py $P/launches_bench_c3.csv > $P/launches_bench_c3_summary.txt
cap() {  # kernel-regex, skip, command...
  local k=$1 s=$2; shift 2
  ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o gpurun_out/r02_$k "$@" \
      > gpurun_out/ncu_$k.log 2>&1 || true
  python profiles/summarize.py gpurun_out/r02_$k.ncu-rep $P/ncu_${k}_c3.txt || true
}
cap score_tc 1 $S
cap select_plan 1 $S
cap select_emit 1 $S
cap budgets 1 $S
cap decode_attn 1 $S
cap kv_project 0 python profiles/kvproj_time.py
ls $P
