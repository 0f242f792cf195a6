# same-box A/B of the model step (n_seq 1, 16): the layer's down GEMV prefetches the next layer's QKV
# weights into L2 in equal per-CTA shares at its start (nx) vs not (base)
L=paper_2605_06676_b200
cp $L/liblkv_b200_nx.so $L/liblkv_b200.so
python -m pytest tests/test_model_decode.py -q -m gpu 2>&1 | tail -1
for r in 1 2; do for v in base nx; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v n1 $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
  echo "$v n16 $(python profiles/model_step_time.py --steps 20 --n-seq 16 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done; done
cp $L/liblkv_b200_nx.so $L/liblkv_b200.so
