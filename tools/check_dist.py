"""Emulated multi-rank evaluate on one GPU vs the single-device evaluate:
uniform, clustered (pruned boxes) and surface clouds, several right-hand
sides, rank counts that do not divide the level-2 boxes evenly."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_07436_b200 import FmmConfig, setup
from paper_2408_07436_b200.distributed import evaluate_local

cases = [
    (dict(depth=4, order_equiv=4, backend="blas", precision="f32", sigma_min=1e-6), 100000, "uniform", 1, (2, 4, 8)),
    (dict(depth=4, order_equiv=4, backend="blas", precision="f64", sigma_min=1e-10), 60000, "uniform", 1, (2, 4, 8)),
    (dict(depth=4, order_equiv=4, backend="fft", precision="f64"), 60000, "uniform", 1, (2, 4, 8)),
    (dict(depth=4, order_equiv=4, backend="blas", precision="f32", sigma_min=1e-6), 60000, "clustered", 2, (3, 5)),
    (dict(depth=5, order_equiv=5, backend="blas", precision="f64", sigma_min=1e-12), 30000, "sphere", 1, (3, 8)),
    (dict(depth=4, order_equiv=6, backend="blas", precision="f64", sigma_min=1e-6), 40000, "clustered", 2, (2, 7)),
    (dict(depth=4, order_equiv=4, backend="fft", precision="f32"), 60000, "clustered", 2, (2, 6)),
    (dict(depth=3, order_equiv=6, backend="blas", precision="f32", sigma_min=1e-6), 20000, "uniform", 1, (2, 3)),
]
worst = 0.0
for kw, n, shape, nrhs, worlds in cases:
    rng = np.random.default_rng(7)
    pts = rng.random((n, 3))
    if shape == "clustered":
        pts = pts ** 3
    elif shape == "sphere":
        v = rng.standard_normal((n, 3))
        pts = (v / np.linalg.norm(v, axis=1)[:, None] + 1) / 2
    q = np.random.default_rng(11).random((n, nrhs)) + 0.1
    inst = setup(pts, pts, FmmConfig(**kw))
    ref = np.asarray(inst.evaluate(q), dtype=np.float64).reshape(n, nrhs)
    for world in worlds:
        got = np.asarray(evaluate_local(inst, world, q), dtype=np.float64)
        rel = np.abs(got - ref) / np.abs(ref)
        tol = 1e-5 if kw["precision"] == "f32" else 1e-10
        worst = max(worst, rel.max() / tol)
        print(kw["backend"], kw["precision"], "p", kw["order_equiv"], shape, "R", nrhs, "world", world,
              "max rel vs 1-GPU", f"{rel.max():.2e}", "OK" if rel.max() <= tol else "FAIL", flush=True)
print("worst / tol", worst)
