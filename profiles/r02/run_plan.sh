timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "select or evict or config3 or config2 or trace" > gpurun_out/plan_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/plan_tests.log
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-sweep --no-decode"
$B > gpurun_out/plan_bench.json 2> gpurun_out/plan_bench.log; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/plan_bench.json').read().splitlines()[-1]);print(d['ms_per_step'],d['stages_ms'])"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"select_plan" -c 5 --csv $B 2>/dev/null | grep select_plan | tail -3
