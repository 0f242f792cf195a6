set -x
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gputest_full.log 2>&1; echo pytest_exit=$?
tail -15 gpurun_out/gputest_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.log; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo ref=$?
