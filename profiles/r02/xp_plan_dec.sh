# plan kernel timing (C3 / C2 / one 8-way shard) + decode with L2 prefetch (model step + all-layer bench decode)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_sharded_gpu.py tests/test_model_decode.py -m gpu -q -x > gpurun_out/pd_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/pd_tests.log
for args in "--config 3" "--config 2" "--config 3 --n-layers 4"; do
  echo "$args: $(ncu --metrics gpu__time_duration.sum --clock-control none -k regex:select_plan -c 3 --csv python profiles/step.py $args --evict 3 --decode 0 2>/dev/null | grep select_plan | awk -F'","' '{print $NF}' | tr '\n' ' ')"
done
python profiles/model_step_time.py --steps 50 > gpurun_out/ms_graph3.json 2> gpurun_out/ms_graph3.log; echo graph=$?; tail -1 gpurun_out/ms_graph3.json
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_attn|decode_combine" --launch-skip 64 --launch-count 64 --csv --log-file gpurun_out/model_launches3.csv python profiles/model_step_time.py --eager --steps 1 > gpurun_out/ms_ncu3.log 2>&1; echo ncu=$?
python profiles/launch_summary.py gpurun_out/model_launches3.csv
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-sweep > gpurun_out/pd_bench.json 2> gpurun_out/pd_bench.log; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/pd_bench.json').read().splitlines()[-1]);print(d['ms_per_step'], d.get('decode',{}).get('ms_per_step'))"
