"""Stress test of the tensor-memory sweep: many small f32 BLAS evaluates
(varying size, depth, order, rhs count) compared with the TMA sweep on the
same instance inputs; reports every mismatch above 1e-5."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_07436_b200 import FmmConfig, setup

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
bad = 0
for it in range(iters):
    n = int(rng.integers(2000, 120000))
    depth = int(rng.integers(3, 6))
    order = int(rng.choice([3, 4]))
    nrhs = int(rng.choice([1, 1, 2]))
    pts = rng.random((n, 3))
    if rng.random() < 0.3:                        # clustered cloud: pruned boxes
        pts = pts ** 3
    q = rng.random((n, nrhs)) if nrhs > 1 else rng.random(n)
    res = {}
    for sweep in ("tma", "tmem"):
        os.environ["KIFMM_F32_SWEEP"] = sweep
        inst = setup(pts, pts, FmmConfig(depth=depth, order_equiv=order, backend="blas",
                                         precision="f32", sigma_min=1e-6))
        res[sweep] = np.asarray(inst.evaluate(q), dtype=np.float64)
        if sweep == "tmem":
            rep = [np.asarray(inst.evaluate(q), dtype=np.float64) for _ in range(3)]
    d = np.abs(res["tmem"] - res["tma"]) / np.abs(res["tma"])
    dr = max(np.abs(r - res["tmem"]).max() for r in rep)
    flag = d.max() > 1e-5 or dr > 0
    bad += flag
    print(f"{it:3d} n={n} depth={depth} p={order} R={nrhs}: max rel {d.max():.2e} repeat diff {dr:.2e}"
          + ("  <-- BAD" if flag else ""), flush=True)
print("bad", bad)
