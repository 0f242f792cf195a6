timeout 900 python -m pytest tests/test_reference_api.py tests/test_policy_io.py tests/test_dropin_cpp.py -m gpu -q > gpurun_out/refapi.log 2>&1; echo exit=$?; tail -30 gpurun_out/refapi.log
