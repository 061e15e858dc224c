"""Run one bench.py extras section alone: python scripts/run_extras.py n4|n1"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2604_15408_b200 as rb
fn = {"n4": bench.n4_general_extras, "n1": bench.n1_block_extras}[sys.argv[1]]
print(json.dumps(fn(rb, torch, torch.device("cuda"), torch.bfloat16), indent=1))
