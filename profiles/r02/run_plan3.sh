timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_sharded_gpu.py -m gpu -q -x > gpurun_out/plan3_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/plan3_tests.log
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-sweep --no-decode"
for c in 3 2; do $B --config $c > gpurun_out/plan3_c$c.json 2> gpurun_out/plan3_c$c.log; echo bench$c=$?
python -c "import json;d=json.loads(open('gpurun_out/plan3_c$c.json').read().splitlines()[-1]);print(d['ms_per_step'],d.get('stages_ms'))"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"select_plan|select_emit|score_tc|budgets" -c 12 --csv $B --config $c 2>/dev/null | grep -E "select_plan|select_emit|score_tc|budgets" | awk -F'","' '{print $5, $NF}' | tail -8; done
