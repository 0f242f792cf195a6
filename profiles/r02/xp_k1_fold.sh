# candidate build (fold = the working tree, e.g. Estrin) vs the committed (v728): parity, then within-box timing
L=paper_2605_06676_b200
cp $L/liblkv_b200_fold.so $L/liblkv_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "score or config3 or evict or kv_project or layerwise" > gpurun_out/fold_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/fold_tests.log
for rep in 1 2 3; do
for v in v728 fold; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v $(python profiles/r02/k1_act.py 2>/dev/null | tail -1)"
done; done
cp $L/liblkv_b200_fold.so $L/liblkv_b200.so
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-sweep --no-decode > gpurun_out/fold_bench.json 2> gpurun_out/fold_bench.log; echo bench=$?
cp $L/liblkv_b200_v728.so $L/liblkv_b200.so
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-sweep --no-decode > gpurun_out/v728_bench.json 2> gpurun_out/v728_bench.log; echo bench=$?
python -c "
import json
for f in ('fold','v728'):
    d=json.loads(open(f'gpurun_out/{f}_bench.json').read().splitlines()[-1]); print(f, d['ms_per_step'], d['value']/1e9)"
