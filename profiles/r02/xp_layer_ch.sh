# same-box A/B of the model step (n_seq 1, 16) and the all-layer decode: the one-wave decode plan sizes
# work items per layer (plch) vs one size for all layers from the busiest layer (base)
L=paper_2605_06676_b200
cp $L/liblkv_b200_plch.so $L/liblkv_b200.so
python -m pytest tests/test_model_decode.py tests/test_gpu_parity.py -q -m gpu -k "decode or model" 2>&1 | tail -2
for r in 1 2; do for v in base plch; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v n1 $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
  echo "$v n16 $(python profiles/model_step_time.py --steps 20 --n-seq 16 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
  echo "$v bench-decode $(python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-sweep 2>/dev/null | tail -1 | grep -o '"decode[^}]*}' | head -c 300)"
done; done
cp $L/liblkv_b200_plch.so $L/liblkv_b200.so
