# within-box headline A/B: the committed build (cur) vs the same tree with the pre-fold score.cu (pf)
L=paper_2605_06676_b200
for r in 1 2 3; do for v in pf cur; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu --no-sweep --no-decode > gpurun_out/fb_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/fb_$v.json').read().splitlines()[-1]);print('$v', round(d['ms_per_step'],4), round(d['stages_ms']['score_K1'],4))"
done; done
cp $L/liblkv_b200_cur.so $L/liblkv_b200.so
