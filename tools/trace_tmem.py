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
names = {0: "g0_have_A", 1: "g0_buf_free", 3: "g0_issue", 4: "stage_free", 5: "g1_have_A", 6: "g1_buf_free"}
rel = np.where(t > 0, t - t0, np.nan)
n = int(np.nanmax(np.where(t[4] > 0, np.arange(1024), -1))) + 1
print("vectors traced", n)
for g in list(range(0, 20)) + list(range(n - 6, n)):
    print(g, " ".join(f"{names[e]}={rel[e][g]:9.0f}" for e in (4, 0, 1, 3, 5, 6)))
iss = rel[3][:n]
iss = iss[~np.isnan(iss)]
print("group-0 issue interval: median %.0f clk (2 vectors per interval)" % np.median(np.diff(iss)))
a0, f0 = rel[0][:n], rel[1][:n]
print("g0 have_A -> buf_free median %.0f; buf_free -> issue median %.0f; stage_free -> have_A median %.0f" % (
    np.nanmedian(f0 - a0), np.nanmedian(rel[3][:n] - f0), np.nanmedian(a0 - rel[4][:n])))
