# K1 epilogue cost at C3: the product build, identity activation (k1), no epilogue math (k2)
L=paper_2605_06676_b200
cp $L/liblkv_b200.so /tmp/lkv_full.so
for v in full k1 k2; do
  if [ $v != full ]; then cp $L/liblkv_b200_$v.so $L/liblkv_b200.so; fi
  echo "$v $(python profiles/r02/k1_act.py 2>/dev/null | tail -1)"
  cp /tmp/lkv_full.so $L/liblkv_b200.so
done
