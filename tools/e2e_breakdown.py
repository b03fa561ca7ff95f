"""Where the public-API evaluate's time goes (config 2): H2D, graph, D2H, host."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2408_07436_b200 import FmmConfig, setup
pts, q = bench.inputs()
inst = setup(pts, pts, FmmConfig(**bench.CONFIG))
qp = torch.from_numpy(q).pin_memory().numpy()
for _ in range(3):
    inst.evaluate(qp)
dev = inst.device
g, static_q, out = dev.graph_for(1)
src = torch.from_numpy(qp).reshape(-1)
print("src pinned:", src.is_pinned())
def t(f, n=20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
print("full evaluate      %.3f ms" % t(lambda: inst.evaluate(qp)))
print("H2D copy           %.3f ms" % t(lambda: static_q.copy_(src)))
print("graph replay       %.3f ms" % t(lambda: g.replay()))
print("D2H .cpu()         %.3f ms" % t(lambda: out.cpu()))
pin = torch.empty(out.shape, dtype=out.dtype).pin_memory()
print("D2H pinned         %.3f ms" % t(lambda: pin.copy_(out)))
print("np copy 4MB        %.3f ms" % t(lambda: pin.numpy().copy()))
print("as_charge_matrix   %.3f ms" % t(lambda: np.ascontiguousarray(qp.reshape(-1, 1), dtype=np.float64)))
