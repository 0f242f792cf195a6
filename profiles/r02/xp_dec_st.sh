# within-box A/B of the model step: per-layer decode ring of 2 stages (st2) vs 3 (st3, committed)
L=paper_2605_06676_b200
for r in 1 2 3; do for v in st2 st3; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done; done
cp $L/liblkv_b200_st3.so $L/liblkv_b200.so
