import os, sys, ctypes
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_07436_b200 import FmmConfig, setup
from paper_2408_07436_b200 import _native as nat

def stuck(tag):
    buf = (ctypes.c_uint * 257)()
    nat.load().kifmm_mbar_debug_read(buf)
    n = buf[0]
    print(tag, "stuck waits", n, flush=True)
    for i in range(min(n, 12)):
        print("   cta", buf[1 + 4*i], "tid", buf[2 + 4*i], "bar smem", buf[3 + 4*i], "parity", buf[4 + 4*i])

g = np.load("tests/golden/eval_blas_f32.npz")
inst = setup(g["points"], g["points"], FmmConfig(depth=3, order_equiv=4, backend="blas", precision="f32", sigma_min=1e-6))
print({l: (p["n_tiles"], p["h"]) for l, p in inst.device.tma_plan.items()}, inst.device.blas.kin)
out = inst.evaluate(g["charges"]); stuck("golden")
rng = np.random.default_rng(3)
for it in range(6):
    n = int(rng.integers(2000, 120000)); depth = int(rng.integers(3, 6)); order = int(rng.choice([3, 4]))
    nrhs = int(rng.choice([1, 1, 2])); pts = rng.random((n, 3))
    if rng.random() < 0.3: pts = pts ** 3
    q = rng.random((n, nrhs)) if nrhs > 1 else rng.random(n)
    inst = setup(pts, pts, FmmConfig(depth=depth, order_equiv=order, backend="blas", precision="f32", sigma_min=1e-6))
    inst.evaluate(q); stuck(f"it{it} n={n} depth={depth} p={order} R={nrhs} kin={inst.device.blas.kin}")
