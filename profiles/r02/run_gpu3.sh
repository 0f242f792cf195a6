set -x
for s in soft_topk policy evictsim model attention; do timeout 300 oracle/_ref/ref_test_$s > gpurun_out/ref_$s.log 2>&1; echo "$s exit=$?"; tail -3 gpurun_out/ref_$s.log; done
