NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --replay-mode range --clock-control none \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  --log-file gpurun_out/final_traffic_range.csv python scripts/r2/traffic_range.py > gpurun_out/final_traffic_range.log 2>&1
cat > /tmp/n4.py <<'PY'
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, bench, paper_2604_15408_b200 as rb
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
print(json.dumps(bench.n4_general_extras(rb, torch, torch.device("cuda", 0), torch.bfloat16)))
PY
timeout 600 python /tmp/n4.py > gpurun_out/final_n4.json 2> gpurun_out/final_n4.err
