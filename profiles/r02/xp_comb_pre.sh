# same-box A/B of the model step: the combine reads each head's length and item range before
# griddepcontrol.wait, lens / tokens_seen advanced by the lm_head GEMV (cb) vs after the wait (new)
L=paper_2605_06676_b200
cp $L/liblkv_b200_cb.so $L/liblkv_b200.so
python -m pytest tests/test_model_decode.py -q -m gpu 2>&1 | tail -1
for r in 1 2 3; do for v in new cb; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done; done
cp $L/liblkv_b200_cb.so $L/liblkv_b200.so
