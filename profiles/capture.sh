#!/bin/bash
# Round capture (run under gpurun):  profiles/capture.sh r01
#  1. plain runs of the commands (must exit 0 before any ncu run)
#  2. launch list of one C2 eviction + decode (cold-cache, serialised: compare shares)
#  3. one `ncu --set full` per hot kernel, summarised into profiles/<round>/
set -e
R=${1:-r01}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out profiles/$R
python profiles/step.py --evict 2 --decode 2 > gpurun_out/plain_step.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file profiles/$R/launches_c2.csv \
    python profiles/step.py --evict 2 --decode 2 > /dev/null 2>&1
for k in score_tc select_emit decode_attn decode_combine; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/${R}_$k \
      python profiles/step.py --evict 2 --decode 2 > gpurun_out/ncu_$k.log 2>&1 || true
  python profiles/summarize.py gpurun_out/${R}_$k.ncu-rep profiles/$R/ncu_$k.txt || true
done
ls profiles/$R
