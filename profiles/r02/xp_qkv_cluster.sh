# same-box A/B of the model step: QKV as a split-K cluster of 2 (q2, 192 CTAs) or 3 (q3, 288 CTAs)
# with the current DSMEM tail vs the group-aligned stream-K (base, 288 CTAs, global fix-up)
L=paper_2605_06676_b200
cp $L/liblkv_b200_q2.so $L/liblkv_b200.so
python -m pytest tests/test_model_decode.py -q -m gpu 2>&1 | tail -1
for r in 1 2; do for v in base q2 q3; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v n1 $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done; done
cp $L/liblkv_b200_base.so $L/liblkv_b200.so
