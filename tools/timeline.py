"""Completion timeline of one overlapped (3-stream) evaluate: every launch's
end event, relative to a start event, grouped by stream (config 2 default)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2408_07436_b200 import FmmConfig, setup, device as D
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
D._TIMELINE = []
t0 = torch.cuda.Event(enable_timing=True)
t0.record()
dev.evaluate_device(qd, 1)
torch.cuda.synchronize()
tl, D._TIMELINE = D._TIMELINE, None
names = {dev.side_stream.cuda_stream: "P2P(low)", dev.hi_stream.cuda_stream: "main(high)"}
names.update({st.cuda_stream: f"M2L{l}(mid)" for l, st in dev.level_streams.items()})
for n, tag, s, e in tl:
    print(f"{t0.elapsed_time(e)*1e3:8.1f} us  {names.get(s, str(s)):10s} {tag:8s} {n}")
