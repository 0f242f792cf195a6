timeout 240 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "kv_project or layerwise or rope" > gpurun_out/kv_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/kv_tests.log
timeout 120 python profiles/kvproj_time.py > gpurun_out/kv_time.json 2> gpurun_out/kv_time.log; echo time=$?; cat gpurun_out/kv_time.json; tail -3 gpurun_out/kv_time.log
