# final validation with the final build (one GPU): GPU tests, the default bench line (C3), C4 / C5
# lines, the reference arm, the model decode step at n_seq 1 / 4 / 16 and its launch list
O=gpurun_out/final2
mkdir -p $O
python -m pytest tests -m gpu -q > $O/gputest.txt 2>&1; echo "gpu tests rc=$?"; tail -2 $O/gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"
python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench rc=$?"
python bench.py --impl reference > $O/bench_ref_c3.json 2> $O/bench_ref_c3.err; echo "ref rc=$?"
for c in 4 5; do python bench.py --config $c --steps 10 --warmup 3 > $O/bench_c$c.json 2> $O/bench_c$c.err; echo "C$c rc=$?"; done
for n in 1 4 16; do python profiles/model_step_time.py --steps 50 --n-seq $n > $O/model_step_n$n.json 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"wstream|decode_attn|decode_combine|embed|gemv" --launch-skip 194 --launch-count 194 --csv --log-file $O/model_launches.csv python profiles/model_step_time.py --eager --steps 1 > $O/ms_ncu.log 2>&1; echo "ncu rc=$?"
python profiles/launch_summary.py $O/model_launches.csv > $O/model_launches_summary.txt 2>&1
