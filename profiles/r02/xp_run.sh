cp paper_2605_06676_b200/liblkv_b200.so /tmp/orig.so
for v in W0 W1 W2 W3 W0 W1; do cp profiles/r02/xp/lib_$v.so paper_2605_06676_b200/liblkv_b200.so; echo "$v $(python profiles/r02/xp_time.py 30 2>/dev/null)"; done
cp /tmp/orig.so paper_2605_06676_b200/liblkv_b200.so
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
