"""Kernel timeline of one graphed evaluate (torch.profiler / CUPTI activity
records: start offset, duration and stream of every kernel), to find the
critical path of the overlapped DAG.
Usage: python tools/timeline.py N "dict(...)" """
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_07436_b200 import FmmConfig, setup

n = int(sys.argv[1]); kw = eval(sys.argv[2])
pts = np.random.default_rng(7).random((n, 3))
q = np.random.default_rng(11).random(n)
inst = setup(pts, pts, FmmConfig(**kw))
dev = inst.device
qd = torch.from_numpy(q).cuda()
for _ in range(3):
    dev.evaluate_graphed(qd, 1)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        dev.evaluate_graphed(qd, 1)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
# split into the three evaluates by gaps; print the last one
groups, cur = [], []
for e in evs:
    if cur and e.time_range.start - max(c.time_range.end for c in cur) > 50:
        groups.append(cur); cur = []
    cur.append(e)
groups.append(cur)
g = groups[-1]
t0 = g[0].time_range.start
end = max(e.time_range.end for e in g)
print(f"evaluates found {len(groups)}; last spans {end - t0:.1f} us, {len(g)} kernels")
for e in g:
    nm = e.name
    for pre in ("void ", "(anonymous namespace)::", "kifmm::"):
        nm = nm.replace(pre, "")
    nm = nm.split("(")[0].split("<")[0][-40:]
    s = e.time_range.start - t0
    print(f"{s:8.1f} {s + e.time_range.elapsed_us():8.1f} {e.time_range.elapsed_us():7.1f}  "
          f"st{getattr(e, 'device_resource_id', -1):>4}  {nm}")
