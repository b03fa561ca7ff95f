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
names = {4: "stage_issued", 0: "have_A", 2: "split_done", 1: "buf_free", 7: "st_done", 3: "issue",
         9: "committed", 8: "promo_wait", 10: "promo_go", 11: "promo_end", 5: "g1_have_A", 6: "g1_buf_free"}
rel = np.where(t > 0, t - t0, np.nan)
n = int(np.nanmax(np.where(t[4] > 0, np.arange(1024), -1))) + 1
print("vectors traced", n)
order = (4, 0, 2, 1, 7, 3, 9, 8, 10, 11)
print("vec " + " ".join(f"{names[e]:>12s}" for e in order))
for g in list(range(0, 40, 2)) + list(range(n - 8, n, 2)):
    print(f"{g:3d} " + " ".join(f"{rel[e][g]:12.0f}" for e in order))
ev = {k: rel[k][:n:2] for k in names}          # group 0 takes the even vectors of an item starting at even g
def med(a, b):
    return np.nanmedian(ev[b] - ev[a])
print("group-0 medians (clk): stage_issued->have_A %.0f | have_A->split_done %.0f | split_done->buf_free %.0f | "
      "buf_free->st_done %.0f | st_done->issue %.0f | issue->committed %.0f" % (
          med(4, 0), med(0, 2), med(2, 1), med(1, 7), med(7, 3), med(3, 9)))
iss = ev[3][~np.isnan(ev[3])]
print("group-0 issue interval median %.0f clk (2 vectors per interval)" % np.median(np.diff(iss)))
bf = ev[1][~np.isnan(ev[1])]
print("issue(v) -> buf_free(v+2) median %.0f clk (MMA completion seen by the group)" % np.nanmedian(ev[1][1:] - ev[3][:-1]))
print("promotion: wait %.0f, tcgen05.ld + adds %.0f" % (np.nanmedian(rel[10] - rel[8]), np.nanmedian(rel[11] - rel[10])))
