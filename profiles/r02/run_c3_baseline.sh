set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --config 3 --ratio 0.15 --steps 20 --warmup 3 > gpurun_out/c3_bench.json 2> gpurun_out/c3_bench.log
echo bench_exit=$?
C="python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu --no-decode"
$C > gpurun_out/c3_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"score|select|budget|flag|decode" -c 60 --csv --log-file gpurun_out/launches_c3.csv $C > gpurun_out/ncu_c3.log 2>&1
echo ncu_exit=$?
