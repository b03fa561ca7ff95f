"""Compare the tcgen05 3xTF32 sweep against the FP32 SIMT sweep and the
oracle on the c2 levels (GPU)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_07436_b200 import FmmConfig, setup
from paper_2408_07436_b200.device import BlasDevice, Linalg, upload_blas_plan, to_dev
from oracle import port

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 4
pts = np.random.default_rng(7).random((n, 3))
inst = setup(pts, pts, FmmConfig(depth=depth, order_equiv=4, backend="blas", precision="f32", sigma_min=1e-6))
ops = inst.blas_ops
la = Linalg("f32")
bt, bs = BlasDevice(ops, np.float32, la, True), BlasDevice(ops, np.float32, la, False)
rng = np.random.default_rng(1)
for lvl in range(2, depth + 1):
    n_s = inst.source_tree.level_keys(lvl).shape[0]; n_t = inst.target_tree.level_keys(lvl).shape[0]
    mult = rng.standard_normal((n_s, 1, ops.s.shape[0])).astype(np.float32)
    plan = upload_blas_plan(inst.blas_plans[lvl])
    out = {}
    for name, bd in (("tc", bt), ("simt", bs)):
        qt = torch.zeros(n_s * bd.kin * 3, dtype=torch.float32, device="cuda")
        acc = torch.zeros(bd.acc_elems(n_t, 1, plan["n_tiles"]), dtype=torch.float32, device="cuda")
        chk = torch.zeros(n_t * bd.n_c, dtype=torch.float32, device="cuda")
        m = to_dev(mult.reshape(n_s, -1))
        bd.run_level(plan, m, n_s, n_t, 1, 1.0, chk, qt, acc)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            bd.run_level(plan, m, n_s, n_t, 1, 1.0, chk, qt, acc)
        torch.cuda.synchronize()
        out[name] = (chk.cpu().numpy().reshape(n_t, -1), (time.perf_counter() - t0) / 5 * 1e3)
    ref = port.apply_level(ops, inst.buckets[lvl], mult, n_t, 1.0)[:, 0]
    sc = np.abs(ref).max()
    print(f"level {lvl}: tc err {np.abs(out['tc'][0]-ref).max()/sc:.2e} ({out['tc'][1]:.3f} ms)  "
          f"simt err {np.abs(out['simt'][0]-ref).max()/sc:.2e} ({out['simt'][1]:.3f} ms)", flush=True)
