"""Emulated multi-rank evaluate on one GPU vs the single-device evaluate."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_07436_b200 import FmmConfig, setup
from paper_2408_07436_b200.distributed import evaluate_local

for kw, n in ((dict(depth=4, order_equiv=4, backend="blas", precision="f32", sigma_min=1e-6), 100000),
              (dict(depth=4, order_equiv=4, backend="blas", precision="f64", sigma_min=1e-10), 60000),
              (dict(depth=4, order_equiv=4, backend="fft", precision="f64"), 60000)):
    pts = np.random.default_rng(7).random((n, 3))
    q = np.random.default_rng(11).random(n)
    inst = setup(pts, pts, FmmConfig(**kw))
    ref = inst.evaluate(q)
    for world in (2, 4, 8):
        got = evaluate_local(inst, world, q)[:, 0]
        rel = np.abs(got - ref) / np.abs(ref)
        print(kw["backend"], kw["precision"], "world", world, "max rel vs 1-GPU", f"{rel.max():.2e}", flush=True)
