mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --tb=line -p no:cacheprovider 2>&1 | tail -45 > gpurun_out/t_pytest.log
