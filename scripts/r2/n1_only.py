import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2604_15408_b200 as rb
dev = torch.device("cuda", 0)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
print(json.dumps(bench.n1_pipeline_extras(rb, torch, dev, torch.bfloat16)), flush=True)
print(json.dumps(bench.n1_block_extras(rb, torch, dev, torch.bfloat16)), flush=True)
