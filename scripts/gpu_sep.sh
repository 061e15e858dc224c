timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/sep_tests.log
timeout 600 python bench.py --steps 500 --warmup 10 --gather-variants none --cpu-seconds 1 --e2e-steps 5 > gpurun_out/sep_bench.json 2> gpurun_out/sep_bench.err
