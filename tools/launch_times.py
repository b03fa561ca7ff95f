"""Per-launch device times (CUDA events) of one c2 evaluate, in order."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2408_07436_b200 import FmmConfig, setup
from paper_2408_07436_b200.device import profile_launches
cfg = dict(bench.CONFIG)
if len(sys.argv) > 1:
    cfg.update(eval(sys.argv[1]))
pts, q = bench.inputs()
inst = setup(pts, pts, FmmConfig(**cfg))
dev = inst.device
qd = torch.from_numpy(q).cuda()
for _ in range(3):
    dev.evaluate_device(qd, 1)
torch.cuda.synchronize()
with profile_launches() as p:
    dev.evaluate_device(qd, 1)
tot = 0
for n, t, ms in p.times():
    tot += ms
    print(f"{t:6s} {n:32s} {ms*1e3:8.1f} us")
print("total", tot)
