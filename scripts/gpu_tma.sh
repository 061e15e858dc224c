RAGGED_TMA_GATHER=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/tma_tests.log
for i in 1 2; do RAGGED_TMA_GATHER=1 timeout 300 python bench.py --steps 2000 --warmup 20 --no-extras --gather-variants none > gpurun_out/tma_$i.json 2>gpurun_out/tma_err.txt; done
timeout 300 python bench.py --steps 2000 --warmup 20 --no-extras --gather-variants none > gpurun_out/notma.json 2>/dev/null
RAGGED_TMA_GATHER=1 timeout 300 python bench.py --steps 1000 --warmup 10 --no-extras --gather-variants none --prune 0.0 > gpurun_out/tma_p0.json 2>/dev/null
