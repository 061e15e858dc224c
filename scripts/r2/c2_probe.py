"""C2 (DeiT-S, B = 32, 12 layers, prune after 4): the bench's two variants --
all layers through the fused path, or the 4 dense layers as ragged_attn on the
padded buffers (cu = b * N) -- and the bitwise/tolerance check of the dense call."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import argparse
import torch
import bench
args = argparse.Namespace(dtype="bf16")
import paper_2604_15408_b200 as rb
dev = torch.device("cuda", 0)
torch.cuda._sleep(400_000_000); torch.cuda.synchronize()
out = bench.config_extras(rb, torch, dev, torch.bfloat16)
print(json.dumps({"C2": out["C2"]}))
