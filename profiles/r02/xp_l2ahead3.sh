# same-box A/B of the model step: L2 prefetch-ahead (4 units) for every GEMV but Wo (nowo, committed) vs
# every GEMV (l2a4) vs none (new)
L=paper_2605_06676_b200
cp $L/liblkv_b200_nowo.so $L/liblkv_b200.so
python -m pytest tests/test_model_decode.py -q -m gpu 2>&1 | tail -1
for r in 1 2 3; do for v in new l2a4 nowo; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done; done
cp $L/liblkv_b200_new.so $L/liblkv_b200.so
