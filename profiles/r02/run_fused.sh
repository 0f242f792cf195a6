timeout 1200 python -m pytest tests/test_model_decode.py tests/test_gpu_parity.py -m gpu -q -x -k "decode or model" > gpurun_out/fused_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/fused_tests.log
python profiles/model_step_time.py --steps 50 > gpurun_out/ms_graph2.json 2> gpurun_out/ms_graph2.log; echo graph=$?; tail -1 gpurun_out/ms_graph2.json
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"wstream|decode_attn|decode_combine|embed|gemv" --launch-skip 162 --launch-count 162 --csv --log-file gpurun_out/model_launches2.csv python profiles/model_step_time.py --eager --steps 1 > gpurun_out/ms_ncu2.log 2>&1; echo ncu=$?
python profiles/launch_summary.py gpurun_out/model_launches2.csv
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-sweep > gpurun_out/fused_bench.json 2> gpurun_out/fused_bench.log; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/fused_bench.json').read().splitlines()[-1]);print(d['ms_per_step'], d.get('decode'))"
