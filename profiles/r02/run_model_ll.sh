python profiles/model_step_time.py --steps 50 > gpurun_out/ms_graph.json 2> gpurun_out/ms_graph.log; echo graph=$?; tail -1 gpurun_out/ms_graph.json
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"wstream|decode_attn|decode_combine|embed|gemv" --launch-skip 194 --launch-count 194 --csv --log-file gpurun_out/model_launches.csv python profiles/model_step_time.py --eager --steps 1 > gpurun_out/ms_ncu.log 2>&1; echo ncu=$?
python profiles/launch_summary.py gpurun_out/model_launches.csv
