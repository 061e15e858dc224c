mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_ws.py -x -q > gpurun_out/j4_pytest_ws.log 2>&1
timeout 600 python scripts/r2/ws_cross.py > gpurun_out/j4_cross.log 2>&1
for c in c3p0 c3p05; do CASE=$c timeout 120 python scripts/r2/ws_tl2.py > gpurun_out/j4_tl_$c.json 2>&1; done
