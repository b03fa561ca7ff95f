"""Generate the golden vectors that pin the oracle and the device path.

Run in the build container, where the reference exists:
    python tests/golden/make_golden.py
It imports the UNMODIFIED reference package (Cython-compiled from
/root/reference by oracle/build_ref.py, i.e. with its compiled _hot loops)
and records inputs + outputs of the hot-path functions at small sizes into
tests/golden/*.npz.  The GPU box never needs /root/reference: tests read
only these files.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import import_reference  # noqa: E402

kifmm3d = import_reference()
from kifmm3d import _hot, engine, hotloops, m2l_blas, m2l_fft, points  # noqa: E402
from kifmm3d.expansion import n_surface  # noqa: E402
from kifmm3d.octree import Domain, Octree  # noqa: E402

assert hotloops.BACKEND == "compiled"


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(a.nbytes for a in map(np.asarray, arrays.values())), "bytes")


def hotloop_fixtures():
    out = {}
    for dt in (np.float32, np.float64):
        tag = np.dtype(dt).name
        rng = np.random.default_rng(100)
        tx, ty, tz = (np.ascontiguousarray(v, dtype=dt) for v in rng.random((3, 60)))
        sx, sy, sz = (np.ascontiguousarray(v, dtype=dt) for v in rng.random((3, 90)))
        sx[:5], sy[:5], sz[:5] = tx[:5], ty[:5], tz[:5]          # coincident pairs -> 0
        q = rng.random((90, 2)).astype(dt)
        pot = np.zeros((60, 2), dtype=dt)
        _hot.laplace_potentials(tx, ty, tz, sx, sy, sz, q, pot, 2)
        mat = np.empty((60, 90), dtype=dt)
        _hot.laplace_matrix(tx, ty, tz, sx, sy, sz, mat, 2)
        # P2P CSR with empty leaves (test_hotloops.py:64-74 style)
        counts_t = rng.integers(1, 8, size=7)
        counts_s = rng.integers(0, 9, size=7)
        counts_s[3] = 0
        lot = np.repeat(np.arange(7, dtype=np.int64), counts_t)
        nt, ns = int(counts_t.sum()), int(counts_s.sum())
        ptx, pty, ptz = (np.ascontiguousarray(v, dtype=dt) for v in rng.random((3, nt)))
        psx, psy, psz = (np.ascontiguousarray(v, dtype=dt) for v in rng.random((3, ns)))
        pq = rng.random((ns, 1)).astype(dt)
        off = np.concatenate([[0], np.cumsum(counts_s)]).astype(np.int64)
        p2p = np.full((nt, 1), 0.5, dtype=dt)                      # accumulate semantics
        _hot.p2p_blocked(ptx, pty, ptz, lot, psx, psy, psz, pq, off, p2p, 2)
        out.update({f"{tag}_tx": tx, f"{tag}_ty": ty, f"{tag}_tz": tz, f"{tag}_sx": sx,
                    f"{tag}_sy": sy, f"{tag}_sz": sz, f"{tag}_q": q, f"{tag}_pot": pot,
                    f"{tag}_mat": mat, f"{tag}_p2p_tx": ptx, f"{tag}_p2p_ty": pty,
                    f"{tag}_p2p_tz": ptz, f"{tag}_p2p_lot": lot, f"{tag}_p2p_sx": psx,
                    f"{tag}_p2p_sy": psy, f"{tag}_p2p_sz": psz, f"{tag}_p2p_q": pq,
                    f"{tag}_p2p_off": off, f"{tag}_p2p_out": p2p})
    for cdt in (np.complex64, np.complex128):
        tag = np.dtype(cdt).name
        rng = np.random.default_rng(101)
        nf, nsc, ntc, nrhs = 9, 3, 4, 2
        khat = (rng.standard_normal((nf, 26, 8, 8)) + 1j * rng.standard_normal((nf, 26, 8, 8))).astype(cdt)
        qhat = (rng.standard_normal((nf, nsc, 8, nrhs)) + 1j * rng.standard_normal((nf, nsc, 8, nrhs))).astype(cdt)
        halo = rng.integers(-1, nsc, size=(ntc, 26)).astype(np.int64)
        phat = np.zeros((nf, ntc, 8, nrhs), dtype=cdt)
        phat[...] = 0.25
        _hot.hadamard_m2l(khat, qhat, halo, phat, 3, 2)
        out.update({f"{tag}_khat": khat, f"{tag}_qhat": qhat, f"{tag}_halo": halo,
                    f"{tag}_phat": phat})
    save("hotloops", **out)


CONFIGS = {
    # name: (n_points, charges kind, FmmConfig kwargs)
    "c1": (10_000, "u01", dict(depth=3, order_equiv=5, backend="blas", precision="f64",
                              sigma_min=1e-12, oversamples=5, seed=0)),
    "blas_f32": (6_000, "u01", dict(depth=3, order_equiv=4, backend="blas", precision="f32",
                                   sigma_min=1e-6)),
    "fft_f64": (6_000, "pm1", dict(depth=3, order_equiv=6, backend="fft", precision="f64")),
    "fft_f32": (5_000, "u01", dict(depth=3, order_equiv=4, backend="fft", precision="f32")),
    "blas_f64_pc": (4_000, "pm1", dict(depth=3, order_equiv=4, order_check=5, backend="blas",
                                      precision="f64", sigma_min=1e-10)),
    "blas_f64_rhs": (3_000, "rhs3", dict(depth=3, order_equiv=4, backend="blas",
                                        precision="f64", sigma_min=1e-9)),
}


def digest(*arrays):
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.int64).tobytes())
    return h.hexdigest()


def charges(kind, n):
    rng = np.random.default_rng(11)
    if kind == "u01":
        return rng.random(n)
    if kind == "pm1":
        return rng.uniform(-1, 1, n)
    if kind == "rhs3":
        return rng.random((n, 3))
    raise ValueError(kind)


def evaluate_fixtures():
    for name, (n, qk, kw) in CONFIGS.items():
        pts = points.generate_points("uniform-cube", n, seed=7)
        q = charges(qk, n)
        inst = engine.setup(pts, pts, engine.FmmConfig(**kw))
        pot = inst.evaluate(q)
        err = inst.relative_error(pot)
        extra = {}
        cfg = inst.config
        lvl = cfg.depth
        side = inst.domain.box_side(lvl)
        mult = inst.multipoles[lvl]
        n_t = inst.target_tree.level_keys(lvl).shape[0]
        if cfg.backend == "blas":
            check = m2l_blas.apply_level(inst.blas_ops, inst.buckets[lvl], mult, n_t,
                                         level_scale=1.0 / side)
            extra = dict(u=inst.blas_ops.u, s=inst.blas_ops.s,
                         ranks=np.array([x.shape[1] for x in inst.blas_ops.ubar]),
                         calls=np.array(inst.m2l_calls))
        else:
            check = m2l_fft.m2l_fft_level(inst.fft_ops, inst.halo_plans[lvl], mult,
                                          level_scale=1.0 / side)
            extra = dict(khat_f0=inst.fft_ops.khat[0], khat_fl=inst.fft_ops.khat[-1],
                         khat_abs_sum=np.abs(inst.fft_ops.khat).sum())
        save("eval_" + name, points=pts, charges=q, potentials=pot, error=np.array(err.error),
             n_excluded=np.array(err.n_excluded), level=np.array(lvl), level_multipoles=mult,
             level_check=check, locals_leaf=inst.locals_[lvl],
             near_sha=np.array(digest(inst._near_idx, inst._near_offsets)),
             **{f"cfg_{k}": np.array(v if v is not None else -1) for k, v in kw.items()
                if not isinstance(v, str)},
             cfg_backend=np.array(kw["backend"]), cfg_precision=np.array(kw["precision"]),
             **extra)


def dense_level_fixture():
    """apply_level / m2l_fft_level on a fully populated level-2 tree against
    dense K_t sums (test_m2l_blas.py:213-248, test_m2l_fft.py:154-171)."""
    order = 4
    pts = np.random.default_rng(8).random((1500, 3))
    dom = Domain(origin=(0.0, 0.0, 0.0), side=1.0 + 1e-9)
    tree = Octree(pts, 2, dom)
    side = dom.box_side(2)
    mult = np.random.default_rng(9).standard_normal((64, 1, n_surface(order)))
    ops = m2l_blas.precompute(order, order, sigma_min=0.0, level_scale=1.0 / side)
    b = m2l_blas.bucket_level(tree, tree, 2)
    blas = m2l_blas.apply_level(ops, b, mult, 64, level_scale=1.0 / side)
    fops = m2l_fft.precompute_fft_operators(order)
    plan = m2l_fft.build_halo_plan(tree, tree, 2)
    fft = m2l_fft.m2l_fft_level(fops, plan, mult, level_scale=1.0 / side)
    save("level2_dense", points=pts, mult=mult, blas=blas, fft=fft, order=np.array(order))


if __name__ == "__main__":
    hotloop_fixtures()
    dense_level_fixture()
    evaluate_fixtures()
