timeout 900 python -m pytest tests/test_gpu_block.py -x -q 2>&1 | tail -3 > gpurun_out/block_tests.log
timeout 600 python scripts/bench_block.py 1248 6304 > gpurun_out/bench_block.json 2> gpurun_out/bench_block.err
