mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prune.py tests/test_gpu_parity.py -q -x -k "evit or topk or prune or mask" 2>&1 | tail -15 > gpurun_out/r2_n2_pytest.log
timeout 300 python scripts/r2/n2_quick.py > gpurun_out/r2_n2_quick.json 2>&1
timeout 300 python scripts/r2/prune_fused_timeline.py > gpurun_out/r2_prune_fused_tl.json 2>&1
timeout 300 python scripts/r2/prune_h_probe.py > gpurun_out/r2_prune_h.json 2>&1
