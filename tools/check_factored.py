"""Factored vs dense float64 BLAS-M2L sweep: same instance inputs, max relative
difference of the potentials, and the level sweep times of both."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_07436_b200 import FmmConfig, setup
from paper_2408_07436_b200.device import profile_launches

cases = [(30000, 4, 5, 1e-12, "uniform", 1), (30000, 5, 5, 1e-12, "sphere", 1),
         (20000, 3, 6, 1e-6, "uniform", 2), (200000, 5, 6, 1e-6, "uniform", 1)]
if len(sys.argv) > 1:
    cases = [eval(sys.argv[1])]
for n, depth, p, sig, shape, nrhs in cases:
    rng = np.random.default_rng(3)
    if shape == "sphere":
        v = rng.standard_normal((n, 3))
        pts = (v / np.linalg.norm(v, axis=1)[:, None] + 1) / 2
    else:
        pts = rng.random((n, 3))
    q = rng.standard_normal((n, nrhs))
    res, times = {}, {}
    for mode in ("dense", "factored"):
        os.environ["KIFMM_F64_SWEEP"] = mode
        inst = setup(pts, pts, FmmConfig(depth=depth, order_equiv=p, backend="blas",
                                         precision="f64", sigma_min=sig))
        res[mode] = inst.evaluate(q)
        dev = inst.device
        qd = torch.from_numpy(q).cuda()
        dev.evaluate_device(qd.reshape(-1), nrhs)
        with profile_launches() as prof:
            dev.evaluate_device(qd.reshape(-1), nrhs)
        t = {}
        for name, tag, ms in prof.times():
            if "sweep" in name or "compress" in name or "expand" in name:
                t[name.replace("kifmm_m2l_", "")] = t.get(name.replace("kifmm_m2l_", ""), 0) + ms
        times[mode] = t
        k, ranks = dev.blas.k, inst.blas_ops.ranks
    d = np.abs(res["factored"] - res["dense"]).max() / np.abs(res["dense"]).max()
    print(f"n={n} depth={depth} p={p} sigma={sig} {shape} R={nrhs}: k={k} mean k_t={ranks.mean():.1f} "
          f"max rel diff {d:.2e}; dense {times['dense']} factored {times['factored']}", flush=True)
