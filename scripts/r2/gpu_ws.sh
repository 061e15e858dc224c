mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ws.py -q -x 2>&1 | tail -25 > gpurun_out/r2_ws_pytest.log
timeout 600 python scripts/r2/ws_quick.py > gpurun_out/r2_ws_quick.txt 2>&1
CASE=vitl timeout 300 python scripts/r2/ws_timeline.py > gpurun_out/r2_ws_tl.json 2>&1
CASE=c3p0 timeout 300 python scripts/r2/ws_timeline.py > gpurun_out/r2_ws_tl_c3.json 2>&1
