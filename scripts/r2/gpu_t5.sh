mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ws.py tests/test_gpu_block.py tests/test_gpu_parity.py -q -rf --tb=short -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/t5_pytest.log
timeout 600 python scripts/r2/ws_cross.py > gpurun_out/t5_cross.log 2>&1
