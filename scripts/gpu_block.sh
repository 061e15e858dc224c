timeout 900 python -m pytest tests/test_gpu_block.py -x -q 2>&1 | tail -5 > gpurun_out/block_tests.log
timeout 600 python scripts/run_extras.py n1 > gpurun_out/n1.json 2> gpurun_out/n1.err
