# within-box A/B of the K1 GELU form: A&S 7.1.28 (committed), 7.1.28 with max(h,0) on the ALU, A&S 7.1.26 scaled
L=paper_2605_06676_b200
cp $L/liblkv_b200.so /tmp/lkv_cur.so
for rep in 1 2 3; do
for v in v728 v728alu v726; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v $(python profiles/r02/k1_act.py 2>/dev/null | tail -1)"
done; done
cp /tmp/lkv_cur.so $L/liblkv_b200.so
