timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > gpurun_out/tc_tests.log
for i in 1 2; do timeout 300 python bench.py --steps 2000 --warmup 20 --no-extras --gather-variants none > gpurun_out/rot_$i.json 2>/dev/null; done
for p in 0.0 0.5; do timeout 300 python bench.py --steps 1000 --warmup 10 --no-extras --gather-variants none --prune $p > gpurun_out/rot_p$p.json 2>/dev/null; done
