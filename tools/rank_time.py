"""Device time of ONE rank's share of the partitioned config-2 evaluate, run
alone on this GPU with the collectives stubbed (distributed.StubCollectives):
the rank's real kernels, row ranges, stream DAG and CUDA graph, without the
NCCL transfers.  Not a multi-GPU measurement - it shows what each GPU of an
N-way run has to do.  Usage: python tools/rank_time.py [worlds, e.g. 2,4,8]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2408_07436_b200 import FmmConfig, setup
from paper_2408_07436_b200 import device as D
from paper_2408_07436_b200.distributed import (DistributedFmm, StubCollectives, make_partition,
                                                make_rank_plans)

worlds = [int(w) for w in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8").split(",")]
pts, q = bench.inputs()
inst = setup(pts, pts, FmmConfig(**bench.CONFIG))
qd = torch.from_numpy(q).cuda()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for world in worlds:
    part = make_partition(inst.source_tree, inst.target_tree, world)
    plans = make_rank_plans(inst, part)
    for rank in sorted({0, world // 2}):
        rk = DistributedFmm(inst, plans[rank], D.DeviceFmm(inst), all_plans=plans)
        coll = StubCollectives(rank)
        for _ in range(3):
            rk.evaluate_graphed(qd, 1, coll)
        ts = []
        for _ in range(20):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rk.evaluate_graphed(qd, 1, coll)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        with D.profile_launches() as prof:
            rk.evaluate(qd, 1, coll)
        agg = {}
        for n, _, t in prof.times():
            agg[n.replace("kifmm_", "")] = agg.get(n.replace("kifmm_", ""), 0.0) + t
        g = rk.halo.groups
        halo_mb = sum(g[k]["smax"] for k in g) * inst.expansions.n_equiv * 4 / 1e6
        top = ", ".join(f"{k} {v * 1e3:.0f}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:6])
        print(f"world {world} rank {rank}: graph median {np.median(ts) * 1e3:.0f} us (min {min(ts) * 1e3:.0f}); "
              f"halo buffer {halo_mb:.2f} MB per rank; eager kernel sums (us): {top}", flush=True)
        del rk
        torch.cuda.empty_cache()
