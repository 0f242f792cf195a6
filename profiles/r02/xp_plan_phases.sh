# plan-kernel phase costs at C3: experiment builds that stop after the prologue (xp3), S2 (xp2), S3 (xp1)
L=paper_2605_06676_b200
cp $L/liblkv_b200.so /tmp/lkv_full.so
for v in xp3 xp2 xp1 full; do
  if [ $v = full ]; then cp /tmp/lkv_full.so $L/liblkv_b200.so; else cp $L/liblkv_b200_$v.so $L/liblkv_b200.so; fi
  echo "$v: $(timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max,sm__cycles_active.min --clock-control none -k regex:select_plan -c 2 --csv python profiles/step.py --config 3 --evict 2 --decode 0 2>/dev/null | grep select_plan | awk -F'","' '{print $(NF-3), $NF}' | tr '\n' ' ')"
done
cp /tmp/lkv_full.so $L/liblkv_b200.so
