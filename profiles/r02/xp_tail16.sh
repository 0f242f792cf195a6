# same-box A/B of the model step at n_seq = 1 and 16: the split-K GEMV tail's inlined residual
# epilogue for any batch (KE = 8 outputs per thread above 2 rows, the 1-output form below) (t16) vs <= 2 rows only (base)
L=paper_2605_06676_b200
cp $L/liblkv_b200_t16.so $L/liblkv_b200.so
python -m pytest tests/test_model_decode.py -q -m gpu 2>&1 | tail -1
for r in 1 2; do for v in base t16; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v n1 $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
  echo "$v n16 $(python profiles/model_step_time.py --steps 20 --n-seq 16 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done; done
cp $L/liblkv_b200_t16.so $L/liblkv_b200.so
