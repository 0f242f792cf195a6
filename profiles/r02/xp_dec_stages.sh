timeout 900 python -m pytest tests/test_model_decode.py tests/test_gpu_parity.py -m gpu -q -x -k "decode or model" > gpurun_out/ds_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/ds_tests.log
python profiles/model_step_time.py --steps 50 > gpurun_out/ds_graph.json 2> gpurun_out/ds_graph.log; echo graph=$?; python -c "import json;print(json.loads(open('gpurun_out/ds_graph.json').read().splitlines()[-1])['ms_per_step'])"
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-sweep > gpurun_out/ds_bench.json 2> gpurun_out/ds_bench.log; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/ds_bench.json').read().splitlines()[-1]);print(d['ms_per_step'], d.get('decode',{}).get('ms_per_step'))"
