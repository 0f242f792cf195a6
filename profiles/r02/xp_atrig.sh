# same-box A/B of the model step (n_seq 1, 16): the attention kernel triggers the combine at its start
# (base) vs at its exit (noat)
L=paper_2605_06676_b200
for r in 1 2; do for v in base noat; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v n1 $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
  echo "$v n16 $(python profiles/model_step_time.py --steps 20 --n-seq 16 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done; done
cp $L/liblkv_b200_base.so $L/liblkv_b200.so
