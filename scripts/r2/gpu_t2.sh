mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gather.py tests/test_gpu_block.py tests/test_gpu_pipeline.py -q -rf --tb=line -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/t2_pytest.log
PROBE_P=0.8,0.0 timeout 300 python scripts/r2/block_breakdown.py > gpurun_out/t2_block.log 2>&1
