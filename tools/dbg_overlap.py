"""Debug: overlapped (multi-stream) evaluate vs sequential, eager and graphed."""
import numpy as np, sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_07436_b200 import FmmConfig, setup
pts = np.random.default_rng(7).random((10000, 3)); q = np.random.default_rng(11).random(10000)
kw = eval(sys.argv[1])
inst = setup(pts, pts, FmmConfig(**kw))
dev = inst.device
qd = torch.from_numpy(q).cuda()
dev.overlap = False
a = dev.evaluate_device(qd, 1).cpu().numpy().copy()
dev.overlap = True
b = dev.evaluate_device(qd, 1).cpu().numpy().copy()
torch.cuda.synchronize()
b2 = dev.evaluate_device(qd, 1).cpu().numpy().copy()
c = dev.evaluate_graphed(qd, 1).cpu().numpy().copy()
r = lambda x: np.abs(x - a).max() / np.abs(a).max()
print("eager-overlap", r(b), "again", r(b2), "graph-overlap", r(c))
