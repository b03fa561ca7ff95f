"""Timeline of CTA 0 of the level-5 brick-fed sweep (config 2)."""
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
dev.evaluate_device(qd, 1)
torch.cuda.synchronize()
nat.call("kifmm_m2l_sweep_tmem_trace", None, 0)
t = buf.cpu().numpy().reshape(12, 1024).astype(np.float64)
t0 = t[t > 0].min()
rel = np.where(t > 0, t - t0, np.nan)
names = {4: "Bslot", 2: "Bissued", 9: "Pstart", 0: "g0A", 1: "g0free", 7: "g0wFull", 3: "g0iss", 5: "g1A", 6: "g1free"}
n = int(np.nanmax(np.where(t[4] > 0, np.arange(1024), -1))) + 1
print("vectors traced", n)
for g in range(0, min(n, 60)):
    print(f"{g:4d} " + " ".join(f"{names[e]}={rel[e][g]:8.0f}" for e in (4, 2, 9, 0, 1, 7, 3, 5, 6)))
kb = rel[8][~np.isnan(rel[8])]
print("brick issue times:", " ".join(f"{x:.0f}" for x in kb[:30]))
iss = rel[3][:n]; iss = iss[~np.isnan(iss)]
print("g0 issue interval median %.0f (2 vectors)" % np.median(np.diff(iss)))
for a, b, nm in ((9, 4, "prod: checks+empty wait"), (4, 2, "prod: B issue"), (0, 1, "wait done"), (1, 7, "free->ready seen"), (7, 3, "issuer wait B full")):
    d = rel[b][:n] - rel[a][:n]
    print(f"{nm:12s} median {np.nanmedian(d):7.0f}  mean {np.nanmean(d):7.0f}")
for a, b, nm in ((1, 10, "free->st done w1"), (1, 11, "free->st done w4"), (10, 7, "w1 stdone->bar")):
    d = rel[b][:n] - rel[a][:n]
    print(f"{nm:18s} median {np.nanmedian(d):7.0f}  mean {np.nanmean(d):7.0f}")
