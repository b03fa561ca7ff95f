"""Timeline of CTA 0 of the level-5 tensor-memory sweep (config 2):
per vector, when the loader had its A row, when its TMEM buffer was free,
when it handed the buffer over, when the MMA issued, when the core stage
was free; per 4-vector block, when the promotion started/finished."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2408_07436_b200 import FmmConfig, setup
from paper_2408_07436_b200 import _native as nat

pts, q = bench.inputs(bench.N_POINTS)
inst = setup(pts, pts, FmmConfig(**bench.CONFIG))
dev = inst.device
qd = torch.from_numpy(q).cuda()
dev.evaluate_device(qd, 1)
torch.cuda.synchronize()
buf = torch.zeros(12 * 1024, dtype=torch.int64, device="cuda")
nat.call("kifmm_m2l_sweep_tmem_trace", buf.data_ptr(), 1 << (inst.config.depth - 1))
# the finest level's sweep runs last among the M2L sweeps in eager order? run
# the level alone through the engine scratch to be sure
b = dev._buffers(1)
lvl = inst.config.depth
mult = None
dev.evaluate_device(qd, 1)
torch.cuda.synchronize()
nat.call("kifmm_m2l_sweep_tmem_trace", None, 0)
t = buf.cpu().numpy().reshape(12, 1024).astype(np.float64)
t0 = t[t > 0].min()
names = ["have_A", "buf_free", "issued", "mma_issue", "stage_free", "promo_start", "promo_end", "x7", "x8", "x9", "x10", "x11"]
n = int((t[3] > 0).sum())
print("vectors traced", n)
rel = np.where(t > 0, t - t0, np.nan)
for g in list(range(0, 24)) + list(range(n - 8, n)):
    print(g, " ".join(f"{names[e]}={rel[e][g]:9.0f}" for e in (0, 1, 3, 2, 4)))
for bc in range(0, 8):
    print("block", bc, f"start={rel[5][bc]:9.0f} end={rel[6][bc]:9.0f}")
d = np.diff(rel[3][:n])
d = np.diff(rel[3][:n])
print("mma issue interval: median %.0f mean %.0f clk" % (np.nanmedian(d), np.nanmean(d)))
print("have_A -> buf_free median %.0f; buf_free -> mma_issue median %.0f; mma_issue -> issued %.0f" % (
    np.nanmedian(rel[1][:n] - rel[0][:n]), np.nanmedian(rel[3][:n] - rel[1][:n]), np.nanmedian(rel[2][:n] - rel[3][:n])))
