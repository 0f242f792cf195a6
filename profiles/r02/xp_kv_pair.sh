# within-box A/B of the K/V projection: 1-SM M=128 kernel vs the 2-SM cta_group::2 kernel
L=paper_2605_06676_b200
for r in 1 2 3; do for v in 1sm 2sm; do
  cp $L/liblkv_b200_$v.so $L/liblkv_b200.so
  python profiles/kvproj_time.py 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$v', round(d['fused_ms'],4), round(d['fused_tflops'],1), round(d['cublas_gemm_ms'],4))"
done; done
cp $L/liblkv_b200_2sm.so $L/liblkv_b200.so
