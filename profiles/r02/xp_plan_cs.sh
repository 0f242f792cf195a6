# A/B of the plan kernel's cluster size (experiment builds liblkv_b200_csX.so, -DLKV_PLAN_CS=X)
cd paper_2605_06676_b200 && cp liblkv_b200.so /tmp/lkv_orig.so && cd ..
for cs in 1 2 4 8; do
  cp paper_2605_06676_b200/liblkv_b200_cs$cs.so paper_2605_06676_b200/liblkv_b200.so
  for c in 3 2; do
    echo "cs=$cs config=$c"
    ncu --metrics gpu__time_duration.sum --clock-control none -k regex:select_plan -c 3 --csv python profiles/step.py --config $c --evict 3 --decode 0 2>/dev/null | grep select_plan | awk -F'","' '{print $NF}' | tr '\n' ' '; echo
  done
done
cp /tmp/lkv_orig.so paper_2605_06676_b200/liblkv_b200.so
ncu --set full --clock-control none --import-source on -k regex:select_plan -s 1 -c 1 -o gpurun_out/r02_plan3 python profiles/step.py --config 3 --evict 2 --decode 0 > gpurun_out/ncu_plan3.log 2>&1; echo ncu=$?
