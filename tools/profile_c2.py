"""One setup + N evaluates of the c2 bench workload (for ncu launch lists
and per-kernel captures: kernels appear in a fixed order per evaluate)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2408_07436_b200 import FmmConfig, setup

n_eval = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = dict(bench.CONFIG)
if len(sys.argv) > 2:
    cfg.update(eval(sys.argv[2]))
n = int(sys.argv[3]) if len(sys.argv) > 3 else bench.N_POINTS
pts, q = bench.inputs(n)
# host setup: the launch list then holds the evaluate's kernels only
inst = setup(pts, pts, FmmConfig(**cfg), device_build=False)
dev = inst.device
qd = torch.from_numpy(q).cuda()
for _ in range(n_eval):
    dev.evaluate_device(qd, 1)
torch.cuda.synchronize()
print("ok", cfg)
