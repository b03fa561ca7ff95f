import numpy as np, sys
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
from conftest import golden
from paper_2408_07436_b200 import setup, FmmConfig
from oracle import port
for name in ["blas_f64_pc", "c1", "blas_f64_rhs"]:
    g = golden("eval_"+name)
    kw = {k[4:]: g[k].item() for k in g.files if k.startswith("cfg_")}
    inst = setup(g["points"], g["points"], FmmConfig(**kw))
    ops = inst.blas_ops
    print(name, "k", ops.k, "golden k", g["u"].shape[1], "u diff", np.abs(ops.u - g["u"]).max() if ops.u.shape == g["u"].shape else "shape!",
          "ranks equal", np.array_equal(ops.ranks, g["ranks"]), "down rank", inst.expansions.down_inv.rank, "up rank", inst.expansions.up_inv.rank)
    pot = port.evaluate(inst, g["charges"]).reshape(g["potentials"].shape)
    want = g["potentials"]
    print("   port vs golden normwise", np.abs(pot - want).max() / np.abs(want).max())
    got = inst.evaluate(g["charges"]).reshape(want.shape)
    print("   gpu vs port normwise", np.abs(got - pot).max() / np.abs(pot).max(), "max rel", (np.abs(got-pot)/np.abs(pot)).max())
