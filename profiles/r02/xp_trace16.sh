# in-graph timeline of the model decode step at n_seq = 16 (instrumented build)
L=paper_2605_06676_b200
cp $L/liblkv_b200.so /tmp/lkv_main.so
cp $L/liblkv_b200_xp.so $L/liblkv_b200.so
python profiles/model_step_time.py --steps 10 --n-seq 16 --trace gpurun_out/trace_step16.npy 2>&1 | tail -2
python profiles/model_step_time.py --steps 10 --trace gpurun_out/trace_step1.npy 2>&1 | tail -2
cp /tmp/lkv_main.so $L/liblkv_b200.so
