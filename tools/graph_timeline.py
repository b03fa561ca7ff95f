"""Operator spans of one graphed config-2 evaluate (external events inside
the graph), in time order: which branch of the DAG ends last."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2408_07436_b200 import FmmConfig, setup
cfg = dict(bench.CONFIG)
if len(sys.argv) > 1:
    cfg.update(eval(sys.argv[1]))
pts, q = bench.inputs()
inst = setup(pts, pts, FmmConfig(**cfg))
dev = inst.device
qd = torch.from_numpy(q).cuda()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(5):
    flush.zero_()
    dev.evaluate_graphed(qd, 1)
torch.cuda.synchronize()
for k, a, b in dev.graph_timeline(1):
    print(f"{k:4s} {a:8.3f} -> {b:8.3f} ms  ({(b - a) * 1e3:7.1f} us)")
