for r in 0 192; do
C="python profiles/model_step_time.py --eager --steps 2 --rows-per-item $r"
$C > /dev/null 2>&1 || { echo plain failed; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_attn|decode_combine|wstream|gemv" -s 200 -c 200 --csv --log-file gpurun_out/dec_launch_$r.csv $C > /dev/null 2>&1
python profiles/launch_summary.py gpurun_out/dec_launch_$r.csv | head -8
done
