# in-graph timeline of the model decode step (experiment build with LKV_XP_TRACE)
L=paper_2605_06676_b200
cp $L/liblkv_b200.so /tmp/lkv_main.so
cp $L/liblkv_b200_xp.so $L/liblkv_b200.so
python profiles/model_step_time.py --steps 20 --trace gpurun_out/trace_step.npy 2>&1 | tail -2
cp /tmp/lkv_main.so $L/liblkv_b200.so
python profiles/model_step_time.py --steps 50 2>&1 | tail -1
