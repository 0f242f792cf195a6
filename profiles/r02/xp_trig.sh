# same-box A/B of the eviction step: K1 and the plan trigger their dependents at their start (trig;
# the plan / emit grids launch early and wait) vs at their exit (base); C3 and C2, 3 alternating reps
L=paper_2605_06676_b200
cp $L/liblkv_b200_trig.so $L/liblkv_b200.so
python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
for r in 1 2 3; do for v in base trig; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v C3 $(python bench.py --no-e2e --no-cpu --no-sweep 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
  echo "$v C2 $(python bench.py --config 2 --no-e2e --no-cpu --no-sweep 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done; done
cp $L/liblkv_b200_trig.so $L/liblkv_b200.so
