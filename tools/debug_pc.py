import numpy as np, sys, torch
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
from conftest import golden
from paper_2408_07436_b200 import setup, FmmConfig
from paper_2408_07436_b200.device import BlasDevice, Linalg, upload_blas_plan, to_dev, sweep_splits
from paper_2408_07436_b200.m2l_blas import dense_cores, level_plan_from_buckets
for name in ["blas_f64_pc", "blas_f64_rhs"]:
    g = golden("eval_"+name)
    kw = {k[4:]: g[k].item() for k in g.files if k.startswith("cfg_")}
    inst = setup(g["points"], g["points"], FmmConfig(**kw))
    lvl = int(g["level"]); mult = g["level_multipoles"][:, :1].copy(); side = inst.domain.box_side(lvl)
    ops = inst.blas_ops; b = inst.buckets[lvl]; n_t = inst.target_tree.level_keys(lvl).shape[0]; n_s = mult.shape[0]
    la = Linalg("f64"); bd = BlasDevice(ops, np.float64, la)
    plan_np = level_plan_from_buckets(b, n_t); plan = upload_blas_plan(plan_np)
    m = to_dev(mult.reshape(n_s, -1))
    qt = torch.zeros(n_s * bd.kin, dtype=torch.float64, device="cuda")
    acc = torch.zeros(bd.acc_elems(n_t, 1, plan["n_tiles"]), dtype=torch.float64, device="cuda")
    check = torch.zeros(n_t * bd.n_c, dtype=torch.float64, device="cuda")
    bd.run_level(plan, m, n_s, n_t, 1, 1/side, check, qt, acc)
    torch.cuda.synchronize()
    qt_np = qt.cpu().numpy().reshape(n_s, bd.kin)
    qref = mult.reshape(n_s, -1) @ ops.s
    print(name, "qt err", np.abs(qt_np[:, :ops.k] - qref).max() / np.abs(qref).max(), "pad max", np.abs(qt_np[:, ops.k:]).max())
    ns = sweep_splits(plan["n_tiles"], bd.n_slabs)
    A = acc.cpu().numpy().reshape(n_t, ns, bd.ko_pad).sum(1)
    D = dense_cores(ops, np.float64)
    from paper_2408_07436_b200.octree import class_transfer_table
    tab = class_transfer_table(); accr = np.zeros((n_t, ops.k))
    for slot, t in enumerate(plan_np.tile_targets):
        if t < 0: continue
        cls = plan_np.tile_class[slot // 128]
        for j in range(189):
            s = plan_np.src[slot, j]
            if s >= 0: accr[t] += D[tab[cls, j]] @ qref[s]
    print(name, "acc err", np.abs(A[:, :ops.k] - accr).max() / np.abs(accr).max(), "acc pad", np.abs(A[:, ops.k:]).max())
    chk = check.cpu().numpy().reshape(n_t, -1)
    cr = (accr @ ops.u.T) / side
    print(name, "check err", np.abs(chk - cr).max() / np.abs(cr).max())
