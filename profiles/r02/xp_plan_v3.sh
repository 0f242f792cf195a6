# A/B of the plan kernel: previous commit (old), new kernel with cs forced 1 / 2, and the default heuristic
L=paper_2605_06676_b200
cp $L/liblkv_b200.so /tmp/lkv_new.so
for v in old cs1 cs2 new; do
  if [ $v = new ]; then cp /tmp/lkv_new.so $L/liblkv_b200.so; else cp $L/liblkv_b200_$v.so $L/liblkv_b200.so; fi
  for args in "--config 3" "--config 2" "--config 3 --n-layers 4"; do
    echo "$v $args: $(ncu --metrics gpu__time_duration.sum --clock-control none -k regex:select_plan -c 3 --csv python profiles/step.py $args --evict 3 --decode 0 2>/dev/null | grep select_plan | awk -F'","' '{print $NF}' | tr '\n' ' ')"
  done
done
cp /tmp/lkv_new.so $L/liblkv_b200.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_sharded_gpu.py -m gpu -q -x > gpurun_out/plan4_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/plan4_tests.log
ncu --set full --clock-control none --import-source on -k regex:select_plan -s 1 -c 1 -o gpurun_out/r02_plan4 python profiles/step.py --config 3 --evict 2 --decode 0 > gpurun_out/ncu_plan4.log 2>&1; echo ncu=$?
