timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gather.py -q 2>&1 | grep -E "FAILED|passed|failed" | head -40 > gpurun_out/tc_tests.log
