# logic check of the N-rank head-sharded bench path on one GPU: every rank on GPU 0, gloo host
# collectives instead of NCCL (bench.py --validate-one-gpu); timings are NOT scaling numbers
for n in 2 4; do
  for pl in lpt layers; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29500 + n)) \
      bench.py --gpus $n --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu --validate-one-gpu --placement $pl \
      > gpurun_out/val_${n}_$pl.json 2> gpurun_out/val_${n}_$pl.log
    echo "n=$n $pl rc=$?"; python -c "import sys,json; d=json.loads(open(\"gpurun_out/val_${n}_$pl.json\").read().splitlines()[-1]); print(d['n_gpus'], d['value'], d.get('parity_gate'), d.get('load_imbalance',{}).get('this_plan_evict'))" 2>&1 | tail -1
  done
done
