timeout 600 python -m pytest tests/test_gpu_gather.py -x -q 2>&1 | tail -15 > gpurun_out/gather_tests.log
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_all.log
