mkdir -p gpurun_out
for c in c3p0 c3p05 c3p08; do CASE=$c timeout 120 python scripts/r2/ws_tl2.py > gpurun_out/j3_tl_$c.json 2>&1; done
PROBE_P=0.8,0.0 timeout 300 python scripts/r2/block_breakdown.py > gpurun_out/j3_block.log 2>&1
