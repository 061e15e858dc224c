timeout 900 python -m pytest tests/test_gpu_block.py -x -q 2>&1 | tail -8 > gpurun_out/block_tests.log
