timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_sharded_gpu.py -m gpu -q -x > gpurun_out/plan5_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/plan5_tests.log
for args in "--config 3" "--config 2" "--config 3 --n-layers 4"; do
  echo "$args: $(ncu --metrics gpu__time_duration.sum --clock-control none -k regex:select_plan -c 3 --csv python profiles/step.py $args --evict 3 --decode 0 2>/dev/null | grep select_plan | awk -F'","' '{print $NF}' | tr '\n' ' ')"
done
ncu --set full --clock-control none --import-source on -k regex:select_plan -s 1 -c 1 -o gpurun_out/r02_plan5 python profiles/step.py --config 3 --evict 2 --decode 0 > gpurun_out/ncu_plan5.log 2>&1; echo ncu=$?
