# same-box A/B of the model step: each GEMV CTA also prefetches into L2 the 4 (l2a4) / 8 (l2a8) weight
# units after its ring's first stages, before griddepcontrol.wait, vs not (new)
L=paper_2605_06676_b200
cp $L/liblkv_b200_l2a4.so $L/liblkv_b200.so
python -m pytest tests/test_model_decode.py -q -m gpu 2>&1 | tail -1
for r in 1 2 3; do for v in new l2a4 l2a8; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done; done
cp $L/liblkv_b200_new.so $L/liblkv_b200.so
