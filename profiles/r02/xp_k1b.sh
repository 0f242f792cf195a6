timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "score or config3 or evict or select" > gpurun_out/k1b_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/k1b_tests.log
python profiles/r02/k1_act.py 2>/dev/null | tail -1
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-sweep --no-decode > gpurun_out/k1b_bench.json 2> gpurun_out/k1b_bench.log; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/k1b_bench.json').read().splitlines()[-1]);print(d['ms_per_step'], d['value']/1e9, d['roofline']['achieved'], d['stages_ms'])"
