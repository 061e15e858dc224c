mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2_base_pytest.log
timeout 300 python scripts/r2/overhead_probe.py > gpurun_out/r2_overhead.json 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_base_bench.json 2> gpurun_out/r2_base_bench.err
echo done > gpurun_out/r2_base_done.txt
