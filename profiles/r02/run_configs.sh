# bench lines at the other BASELINE configs (C4: 16 ragged sequences; C5: Llama-3-70B shape, 640 skewed logits)
for c in 4 5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu --no-sweep > gpurun_out/cfg$c.json 2> gpurun_out/cfg$c.log
  echo "C$c rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/cfg$c.json').read().splitlines()[-1]);print(d['config']['workload'], d['ms_per_step'], d['value']/1e9, d['roofline']['frac'], d.get('step_roofline'), d.get('decode',{}).get('ms_per_step'), d.get('decode',{}).get('frac_of_measured_hbm'))"
done
