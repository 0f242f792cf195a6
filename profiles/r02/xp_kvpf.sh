# same-box A/B of the model step (n_seq 1, 4) and all-layer decode: each attention item prefetches its K/V rows past the ring into L2 before its first ring wait (kvpf) vs not (base)
L=paper_2605_06676_b200
cp $L/liblkv_b200_kvpf.so $L/liblkv_b200.so
python -m pytest tests/test_model_decode.py -q -m gpu 2>&1 | tail -1
for r in 1 2; do for v in base kvpf; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  echo "$v n1 $(python profiles/model_step_time.py --steps 50 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
  echo "$v bench-decode $(python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-sweep 2>/dev/null | tail -1 | grep -o "\"decode\": {[^,]*, \"ms_per_step\": [0-9.]*")"
  echo "$v n4 $(python profiles/model_step_time.py --steps 30 --n-seq 4 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')"
done; done
cp $L/liblkv_b200_kvpf.so $L/liblkv_b200.so
