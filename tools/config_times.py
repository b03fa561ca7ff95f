"""Device evaluate time + per-phase breakdown for a BASELINE-style config."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_07436_b200 import FmmConfig, setup
from paper_2408_07436_b200.device import profile_launches

n = int(sys.argv[1]); kw = eval(sys.argv[2]); mode = sys.argv[3] if len(sys.argv) > 3 else ""
if "sphere" in mode:       # BASELINE config 5: unit-sphere surface scaled into [0,1]^3, N(0,1)
    g = np.random.default_rng(7).standard_normal((n, 3))
    pts = (g / np.linalg.norm(g, axis=1, keepdims=True) + 1.0) / 2.0
    q = np.random.default_rng(11).standard_normal(n)
else:
    pts = np.random.default_rng(7).random((n, 3))
    rng = np.random.default_rng(11)
    q = rng.uniform(-1, 1, n) if "signed" in mode else rng.random(n)
t0 = time.perf_counter(); inst = setup(pts, pts, FmmConfig(**kw)); ts = time.perf_counter() - t0
dev = inst.device
qd = torch.from_numpy(q).cuda()
grad = "grad" in mode
for _ in range(2):
    dev.evaluate_graphed(qd, 1, gradient=grad)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    dev.evaluate_graphed(qd, 1, gradient=grad)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
with profile_launches() as p:
    dev.evaluate_device(qd, 1, gradient=grad)
agg = {}
for name, tag, t in p.times():
    key = tag[:3] + ":" + name.replace("kifmm_", "")
    agg[key] = agg.get(key, 0) + t
print(f"n={n} {kw} {mode} setup {ts:.1f}s evaluate {ms:.3f} ms -> {n/ms/1e3:.1f} Mpts/s")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:12]:
    print(f"   {k:40s} {v*1e3:9.1f} us")
for name, tag, t in p.times():
    if "m2l_sweep" in name:
        print(f"   sweep {tag:10s} {name:32s} {t*1e3:9.1f} us")
