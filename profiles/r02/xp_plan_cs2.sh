L=paper_2605_06676_b200
cp $L/liblkv_b200.so /tmp/lkv_full.so
for v in cs2 cs4 full; do
  if [ $v = full ]; then cp /tmp/lkv_full.so $L/liblkv_b200.so; else cp $L/liblkv_b200_$v.so $L/liblkv_b200.so; fi
  for args in "--config 3" "--config 2"; do
  echo "$v $args: $(timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:select_plan -c 3 --csv python profiles/step.py $args --evict 3 --decode 0 2>/dev/null | grep select_plan | awk -F'","' '{print $NF}' | tr '\n' ' ')"
  done
done
cp /tmp/lkv_full.so $L/liblkv_b200.so
