# in-graph cost of the per-layer attention + combine in the model step: the product build vs an
# experiment build that skips those launches (outputs invalid, timing only)
L=paper_2605_06676_b200
cp $L/liblkv_b200.so /tmp/lkv_cur.so
for rep in 1 2; do
  cp $L/liblkv_b200_m2.so $L/liblkv_b200.so; echo "no_combine $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o "\"ms_per_step\": [0-9.]*")"
  cp /tmp/lkv_cur.so $L/liblkv_b200.so; echo "full $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
  cp $L/liblkv_b200_m1.so $L/liblkv_b200.so; echo "no_attn $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done
cp /tmp/lkv_cur.so $L/liblkv_b200.so
