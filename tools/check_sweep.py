"""Compare the f32 evaluate with the tensor-memory sweep against the TMA sweep
(same process, same inputs) for a few tree shapes; prints the max relative
difference per configuration."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_07436_b200 import FmmConfig, setup

cases = [("golden", 3, 4), (20000, 3, 4), (60000, 4, 4), (200000, 5, 4), (3000, 3, 4), (20000, 3, 3)]
for n, depth, order in cases:
    if n == "golden":
        g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                 "tests", "golden", "eval_blas_f32.npz"))
        pts, q = g["points"], g["charges"]
    else:
        pts = np.random.default_rng(7).random((n, 3))
        q = np.random.default_rng(11).random(n)
    res = {}
    for sweep in ("tma", "tmem"):
        os.environ["KIFMM_F32_SWEEP"] = sweep
        inst = setup(pts, pts, FmmConfig(depth=depth, order_equiv=order, backend="blas",
                                         precision="f32", sigma_min=1e-6))
        res[sweep] = inst.evaluate(q).astype(np.float64)
        k = inst.device.blas.k
    d = np.abs(res["tmem"] - res["tma"]) / np.abs(res["tma"])
    print(f"n={n} depth={depth} p={order} k={k}: max rel diff {d.max():.3e}", flush=True)
    # repeat the tmem evaluate: nondeterminism shows as a difference
    for rep in range(3):
        again = inst.evaluate(q).astype(np.float64)
        print(f"   repeat {rep}: max rel diff vs first {np.abs(again - res['tmem']).max() / np.abs(res['tmem']).max():.3e}", flush=True)
