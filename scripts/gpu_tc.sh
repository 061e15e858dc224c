timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/tc_tests.log
for p in 0.0 0.5 0.8; do timeout 300 python bench.py --steps 1000 --warmup 10 --no-extras --gather-variants none --engine 1 --prune $p > gpurun_out/b_mma_$p.json 2>/dev/null; done
