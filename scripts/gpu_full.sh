timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_all.log
timeout 1200 python bench.py --steps 2000 --warmup 20 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
