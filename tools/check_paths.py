"""Bitwise agreement of the evaluate paths on one instance (GPU): public
evaluate (graph), graph with gradient, eager overlapped, eager sequential."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_07436_b200 import FmmConfig, setup

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
kw = eval(sys.argv[2]) if len(sys.argv) > 2 else dict(depth=5, order_equiv=8, backend="fft",
                                                      precision="f64")
pts = np.random.default_rng(7).random((n, 3))
q = np.random.default_rng(11).uniform(-1, 1, n)
inst = setup(pts, pts, FmmConfig(**kw))
dev = inst.device
a = np.asarray(inst.evaluate(q), np.float64)
qd = torch.from_numpy(q).cuda()
g_pot, g_grad = dev.evaluate_graphed(qd, 1, gradient=True)
b = g_pot.cpu().numpy()[:, 0].astype(np.float64)
c = dev.evaluate_device(qd, 1, timings=True).cpu().numpy()[:, 0].astype(np.float64)
d = dev.evaluate_device(qd, 1).cpu().numpy()[:, 0].astype(np.float64)
e = np.asarray(inst.evaluate(q), np.float64)
sc = np.abs(a).max()
for name, v in (("graph+gradient", b), ("eager sequential", c), ("eager overlapped", d),
                ("public again", e)):
    diff = np.abs(v - a)
    print(f"{name:18s} bitwise {np.array_equal(v, a)}  max|d|/||phi|| {diff.max() / sc:.3e}  "
          f"floored {(diff / np.maximum(np.abs(a), 1e-3 * sc)).max():.3e}")
