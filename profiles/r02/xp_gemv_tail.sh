# same-box A/B of the model step: split-K GEMV tail (live-column DSMEM reduce with all peer loads in
# flight, inlined residual epilogue, split cluster arrive/wait) -- new vs base (the committed build);
# then the in-graph timeline of the new build (LKV_XP_TRACE experiment build)
L=paper_2605_06676_b200
cp $L/liblkv_b200_new.so $L/liblkv_b200.so
python -m pytest tests/test_model_decode.py -q -m gpu 2>&1 | tail -1
for r in 1 2 3; do for v in base new; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done; done
cp $L/liblkv_b200_xp.so $L/liblkv_b200.so
python profiles/model_step_time.py --steps 20 --trace gpurun_out/trace_step.npy 2>&1 | tail -1 | cut -c1-100
cp $L/liblkv_b200_new.so $L/liblkv_b200.so
