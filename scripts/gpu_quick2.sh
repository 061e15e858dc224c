for i in 1 2; do timeout 300 python bench.py --steps 2000 --warmup 20 --no-extras --gather-variants none > gpurun_out/q_$i.json 2>/dev/null; done
timeout 300 python bench.py --steps 1000 --warmup 10 --no-extras --gather-variants none --prune 0.0 > gpurun_out/q_p0.json 2>/dev/null
