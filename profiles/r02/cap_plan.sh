S="python profiles/step.py --config 3 --evict 2 --decode 0"
$S > gpurun_out/plain_step.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:select_plan -s 1 -c 1 -o gpurun_out/r02_plan2 $S > gpurun_out/ncu_plan2.log 2>&1
echo ncu=$?
