# within-box A/B of the K1 GELU epilogue's FP32 instruction form: packed FFMA2 pairs (committed),
# half packed / half scalar (s1), all scalar (s2)
L=paper_2605_06676_b200
cp $L/liblkv_b200.so /tmp/lkv_cur.so
for rep in 1 2 3; do
for v in cur s1 s2; do
  if [ $v = cur ]; then cp /tmp/lkv_cur.so $L/liblkv_b200.so; else cp $L/liblkv_b200_$v.so $L/liblkv_b200.so; fi
  echo "$v $(python profiles/r02/k1_act.py 2>/dev/null | tail -1)"
done; done
cp /tmp/lkv_cur.so $L/liblkv_b200.so
