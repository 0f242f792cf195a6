C="python profiles/model_step_time.py --eager --steps 2 --rows-per-item 0"
$C > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"decode_attn" -s 40 -c 1 -o gpurun_out/r02_deccl $C > gpurun_out/ncu_deccl.log 2>&1
echo ncu=$?
