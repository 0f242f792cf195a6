timeout 900 python -m pytest tests/test_model_decode.py tests/test_gpu_parity.py -m gpu -q -x -k "decode or model" > gpurun_out/cb_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/cb_tests.log
for r in 1 2; do
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-sweep > gpurun_out/cb_bench.json 2> gpurun_out/cb_bench.log
python -c "import json;d=json.loads(open('gpurun_out/cb_bench.json').read().splitlines()[-1]);print('decode', d['decode']['ms_per_step'])"
python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*'
done
