for c in "1248 2304 768 0" "1248 768 3072 2" "1248 3072 768 1"; do timeout 120 python scripts/gemm_probe.py $c; done > gpurun_out/gemm_probe.txt 2>&1
timeout 600 python scripts/bench_block.py 1248 6304 50000 > gpurun_out/bench_block.json 2> gpurun_out/bench_block.err
