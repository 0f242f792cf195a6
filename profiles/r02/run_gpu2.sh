# round-2 check: GPU tests, the C3 headline bench, the head-sharded path at N=1
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gputest.log 2>&1
echo pytest_exit=$?
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.log
echo bench_exit=$?
timeout 600 python bench.py --sharded-path --steps 10 --warmup 3 > gpurun_out/bench_sh1.json 2> gpurun_out/bench_sh1.log
echo sharded_exit=$?
