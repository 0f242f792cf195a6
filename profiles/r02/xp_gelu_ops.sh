# K1 time vs the GELU's FMA-pipe op count (experiment builds: g1 -3 FMUL2, g2 -3 FFMA2, g3 both); 3 repeats each
L=paper_2605_06676_b200
cp $L/liblkv_b200.so /tmp/lkv_full.so
for rep in 1 2 3; do
for v in full g1 g2 g3; do
  if [ $v != full ]; then cp $L/liblkv_b200_$v.so $L/liblkv_b200.so; fi
  echo "$v $(python profiles/r02/k1_act.py 2>/dev/null | tail -1)"
  cp /tmp/lkv_full.so $L/liblkv_b200.so
done; done
