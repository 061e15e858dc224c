for c in "1248 2304 768 0" "1248 768 3072 2" "6304 2304 768 0" "50000 2304 768 0"; do timeout 120 python scripts/gemm_probe.py $c; done > gpurun_out/gemm_probe.txt 2>&1
