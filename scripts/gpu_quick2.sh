for i in 1 2; do RAGGED_LIB=paper_2604_15408_b200/libragged_culate.so timeout 300 python bench.py --steps 2000 --warmup 20 --no-extras --gather-variants none > gpurun_out/cul_$i.json 2>/dev/null; done
RAGGED_LIB=paper_2604_15408_b200/libragged_culate.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cu" 2>&1 | tail -2 > gpurun_out/q_tests.log
timeout 300 python bench.py --steps 2000 --warmup 20 --no-extras --gather-variants none > gpurun_out/cu_1.json 2>/dev/null
