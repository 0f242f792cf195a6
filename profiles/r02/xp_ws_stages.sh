# same-box A/B of the model step (n_seq 1, 4): GEMV ring of 5 stages for one batch tile (ws5) vs 4 (ws4)
L=paper_2605_06676_b200
cp $L/liblkv_b200_ws5.so $L/liblkv_b200.so
python -m pytest tests/test_model_decode.py -q -m gpu 2>&1 | tail -1
for r in 1 2; do for v in ws4 ws5; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v n1 $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
  echo "$v n4 $(python profiles/model_step_time.py --steps 30 --n-seq 4 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done; done
cp $L/liblkv_b200_ws5.so $L/liblkv_b200.so
