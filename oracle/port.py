"""ORACLE - test infrastructure only.  Imported by tests/, by
``__graft_entry__.smoke()`` (as the checker) and by ``bench.py``'s CPU
baseline leg; never by the product package.

CPU restatement of the reference's evaluate path (``pkg/src/kifmm3d``),
operating on the host plan of a :class:`paper_2408_07436_b200.FmmInstance`
(trees, operators and per-level plans, which tests/test_setup_parity.py pins
bit-for-bit against the reference's own setup).  The inner loops call the C
restatement in ``oracle/hot.c`` (bit-identical to ``_hot.pyx`` with the same
compiler flags) or, when that library is not built, NumPy twins of
``_hot_fallback.py``.

Parity pinning: tests/test_oracle_golden.py checks every function here
against golden vectors produced by the reference itself
(tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

INV_4PI = 0.079577471545947667884441881686257181
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "_build", "libkifmm_oracle.so")
_lib = None


def _load():
    global _lib
    if _lib is None and os.path.exists(_LIB):
        _lib = ctypes.CDLL(_LIB)
    return _lib


def _threads(threads):
    return int(threads) if threads else (os.cpu_count() or 1)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _suffix(dt):
    return "f32" if np.dtype(dt) == np.float32 else "f64"


# ------------------------------------------------------------------ hot loops
def _weights(tx, ty, tz, sx, sy, sz):
    """_hot_fallback.py:16-27."""
    dx = tx[:, None] - sx[None, :]
    dy = ty[:, None] - sy[None, :]
    dz = tz[:, None] - sz[None, :]
    r2 = dx * dx
    r2 += dy * dy
    r2 += dz * dz
    np.sqrt(r2, out=r2)
    with np.errstate(divide="ignore"):
        w = np.array(r2.dtype.type(INV_4PI), dtype=r2.dtype) / r2
    w[r2 == 0] = 0
    return w


def laplace_potentials(tx, ty, tz, sx, sy, sz, q, out, threads=None):
    """_hot.pyx:24-65: out[i, r] += sum_j K(t_i, s_j) q[j, r]."""
    lib = _load()
    nt, ns = tx.shape[0], sx.shape[0]
    if nt == 0 or ns == 0:
        return out
    if lib is not None:
        dt = tx.dtype
        fn = getattr(lib, "oracle_laplace_potentials_" + _suffix(dt))
        args = [np.ascontiguousarray(a, dtype=dt) for a in (tx, ty, tz, sx, sy, sz)]
        qq = np.ascontiguousarray(q, dtype=dt)
        assert out.flags.c_contiguous and out.dtype == dt
        fn(_p(args[0]), _p(args[1]), _p(args[2]), ctypes.c_int64(nt), _p(args[3]), _p(args[4]),
           _p(args[5]), ctypes.c_int64(ns), _p(qq), ctypes.c_int64(qq.shape[1]), _p(out),
           ctypes.c_int(_threads(threads)))
        return out
    w = _weights(tx, ty, tz, sx, sy, sz)
    for r in range(q.shape[1]):
        out[:, r] += w @ q[:, r]
    return out


def laplace_matrix(tx, ty, tz, sx, sy, sz, threads=None):
    """_hot.pyx:68-88."""
    lib = _load()
    dt = tx.dtype
    out = np.empty((tx.shape[0], sx.shape[0]), dtype=dt)
    if lib is not None and out.size:
        fn = getattr(lib, "oracle_laplace_matrix_" + _suffix(dt))
        a = [np.ascontiguousarray(v, dtype=dt) for v in (tx, ty, tz, sx, sy, sz)]
        fn(_p(a[0]), _p(a[1]), _p(a[2]), ctypes.c_int64(tx.shape[0]), _p(a[3]), _p(a[4]),
           _p(a[5]), ctypes.c_int64(sx.shape[0]), _p(out), ctypes.c_int(_threads(threads)))
        return out
    out[...] = _weights(tx, ty, tz, sx, sy, sz)
    return out


def p2p_blocked(tx, ty, tz, leaf_of_target, sx, sy, sz, q, src_offsets, out, threads=None):
    """_hot.pyx:91-138 (gathered-source CSR form)."""
    lib = _load()
    nt = tx.shape[0]
    if lib is not None and nt:
        dt = tx.dtype
        fn = getattr(lib, "oracle_p2p_blocked_" + _suffix(dt))
        a = [np.ascontiguousarray(v, dtype=dt) for v in (tx, ty, tz, sx, sy, sz)]
        qq = np.ascontiguousarray(q, dtype=dt)
        lot = np.ascontiguousarray(leaf_of_target, dtype=np.int64)
        off = np.ascontiguousarray(src_offsets, dtype=np.int64)
        fn(_p(a[0]), _p(a[1]), _p(a[2]), ctypes.c_int64(nt), _p(lot), _p(a[3]), _p(a[4]), _p(a[5]),
           _p(qq), ctypes.c_int64(qq.shape[1]), _p(off), _p(out), ctypes.c_int(_threads(threads)))
        return out
    bounds = np.searchsorted(leaf_of_target, np.arange(src_offsets.shape[0]))
    for b in range(src_offsets.shape[0] - 1):
        i0, i1 = bounds[b], bounds[b + 1]
        j0, j1 = src_offsets[b], src_offsets[b + 1]
        if i0 < i1 and j0 < j1:
            laplace_potentials(tx[i0:i1], ty[i0:i1], tz[i0:i1], sx[j0:j1], sy[j0:j1], sz[j0:j1],
                               q[j0:j1], out[i0:i1])
    return out


def hadamard_m2l(khat, qhat, halo, phat, threads=None):
    """_hot.pyx:141-178: phat[f,c,t,r] += sum_o sum_s khat[f,o,t,s] qhat[f,halo[c,o],s,r]."""
    lib = _load()
    if lib is not None and phat.size:
        fn = getattr(lib, "oracle_hadamard_m2l_" + ("c64" if khat.dtype == np.complex64 else "c128"))
        k = np.ascontiguousarray(khat)
        q = np.ascontiguousarray(qhat)
        h = np.ascontiguousarray(halo, dtype=np.int64)
        assert phat.flags.c_contiguous
        fn(_p(k), _p(q), _p(h), _p(phat), ctypes.c_int64(k.shape[0]), ctypes.c_int64(q.shape[1]),
           ctypes.c_int64(h.shape[0]), ctypes.c_int64(q.shape[3]), ctypes.c_int(_threads(threads)))
        return phat
    for o in range(26):
        src = halo[:, o]
        hit = np.flatnonzero(src >= 0)
        if hit.size:
            phat[:, hit] += khat[:, o][:, None] @ qhat[:, src[hit]]
    return phat


# ------------------------------------------------------------- level passes
def _expand_rows(rows, n_rhs):
    """m2l_blas.py:264-267."""
    if n_rhs == 1:
        return rows
    return (rows[:, None] * n_rhs + np.arange(n_rhs)[None, :]).ravel()


def apply_level(ops, buckets, multipoles, n_targets, level_scale=1.0):
    """m2l_blas.apply_level, serial strategy (m2l_blas.py:270-326)."""
    n_src, n_rhs, n_e = multipoles.shape
    dtype = multipoles.dtype
    qt = multipoles.reshape(n_src * n_rhs, n_e) @ ops.s
    acc = np.zeros((n_targets * n_rhs, ops.k), dtype=dtype)
    for i, pr in enumerate(buckets.pairs):
        if pr is None or ops.ubar[i].shape[1] == 0:
            continue
        rows_s, rows_t = pr
        g = qt[_expand_rows(rows_s, n_rhs)]
        acc[_expand_rows(rows_t, n_rhs)] += (g @ ops.vbar[i]) @ ops.ubar[i].T
    check = (acc @ ops.u.T) * dtype.type(level_scale)
    return check.reshape(n_targets, n_rhs, ops.u.shape[0])


def m2l_fft_level(ops, plan, multipoles, level_scale=1.0, workers=None):
    """m2l_fft.m2l_fft_level (m2l_fft.py:218-261)."""
    import scipy.fft
    n_src, n_rhs, n_e = multipoles.shape
    grid = ops.grid
    n = grid.n_grid
    dtype = multipoles.dtype
    cdt = np.complex64 if dtype == np.float32 else np.complex128
    w = _threads(workers)
    grids = np.zeros((n_src * n_rhs, n ** 3), dtype=dtype)
    grids[:, grid.embed_idx] = multipoles.reshape(n_src * n_rhs, n_e)
    qhat = scipy.fft.rfftn(grids.reshape(-1, n, n, n), axes=(1, 2, 3), workers=w)
    qhat = qhat.reshape(n_src, n_rhs, grid.n_freq).astype(cdt, copy=False)
    qcl = np.zeros((plan.n_src_clusters * 8, n_rhs, grid.n_freq), dtype=cdt)
    qcl[plan.src_slot] = qhat
    qcl = np.ascontiguousarray(qcl.reshape(plan.n_src_clusters, 8, n_rhs, grid.n_freq)
                               .transpose(3, 0, 1, 2))
    phat = np.zeros((grid.n_freq, plan.n_tgt_clusters, 8, n_rhs), dtype=cdt)
    hadamard_m2l(ops.khat, qcl, plan.halo, phat, threads=workers)
    n_tgt = plan.tgt_slot.shape[0]
    spectra = phat.transpose(1, 2, 3, 0).reshape(plan.n_tgt_clusters * 8, n_rhs,
                                                 grid.n_freq)[plan.tgt_slot]
    pot = scipy.fft.irfftn(spectra.reshape(-1, n, n, n // 2 + 1), s=(n, n, n), axes=(1, 2, 3),
                           workers=w)
    check = pot.reshape(n_tgt * n_rhs, n ** 3)[:, grid.read_idx]
    check = check.astype(dtype, copy=False) * dtype.type(level_scale)
    return check.reshape(n_tgt, n_rhs, n_e)


def _solve(inv, phi, scale):
    """expansion.RegularizedInverse.apply (expansion.py:78-82), column block."""
    return (inv.v @ (inv.inv_vals[:, None] * (inv.u.T @ phi))) * scale


# -------------------------------------------------------------- full evaluate
def evaluate(inst, charges, threads=None, timings=None, state=None):
    """engine.evaluate (engine.py:270-404) on the product's host plan.

    Returns potentials in the caller's target order, in the working dtype.
    ``timings`` (dict) receives per-operator wall seconds like the reference;
    ``state`` (dict) receives the per-level ``multipoles`` and ``locals``.
    """
    import time

    from paper_2408_07436_b200.engine import as_charge_matrix, leaf_centers, leaf_surface_base

    cfg = inst.config
    dtype = np.dtype(cfg.dtype)
    st, tt = inst.source_tree, inst.target_tree
    exp = inst.expansions
    n_e, n_c = exp.n_equiv, exp.n_check
    q = as_charge_matrix(np.asarray(charges), st.n_points).astype(np.float64)
    n_rhs = q.shape[1]
    q_tree = np.ascontiguousarray(q[st.perm], dtype=dtype)
    depth = cfg.depth
    tm = {} if timings is None else timings
    sx, sy, sz = (np.ascontiguousarray(v, dtype=dtype) for v in (st.x, st.y, st.z))
    tx, ty, tz = (np.ascontiguousarray(v, dtype=dtype) for v in (tt.x, tt.y, tt.z))
    leaf_side = inst.domain.box_side(depth)

    # P2M (engine.py:298-319): per leaf, check-surface potentials then up_inv solve.
    from paper_2408_07436_b200.octree import child_index_codes, parent_codes
    t0 = time.perf_counter()
    mult = [np.zeros((st.level_keys(l).shape[0], n_rhs, n_e), dtype=dtype)
            for l in range(depth + 1)]
    checks = np.ascontiguousarray(
        leaf_centers(st)[:, None, :] + leaf_surface_base(cfg.resolved_order_check(), leaf_side,
                                                         cfg.outer_scale)[None], dtype=dtype)
    nl = st.leaves.shape[0]
    # sibling-set blocks of p2m_block sets (engine.py:302-304)
    prow_leaf = np.searchsorted(st.level_keys(depth - 1), parent_codes(st.leaves))
    set_starts = np.flatnonzero(np.r_[True, prow_leaf[1:] != prow_leaf[:-1]])
    block_starts = np.r_[set_starts[::max(1, cfg.p2m_block)], nl]
    for b0, b1 in zip(block_starts[:-1], block_starts[1:]):
        phi = np.empty((b1 - b0, n_rhs, n_c), dtype=dtype)
        for i in range(b0, b1):
            s0 = int(st.leaf_starts[i])
            s1 = s0 + int(st.leaf_counts[i])
            g = checks[i]
            o = np.zeros((n_c, n_rhs), dtype=dtype)
            laplace_potentials(np.ascontiguousarray(g[:, 0]), np.ascontiguousarray(g[:, 1]),
                               np.ascontiguousarray(g[:, 2]), sx[s0:s1], sy[s0:s1], sz[s0:s1],
                               q_tree[s0:s1], o, threads)
            phi[i - b0] = o.T
        nb = b1 - b0
        mult[depth][b0:b1] += _solve(exp.up_inv, phi.reshape(nb * n_rhs, n_c).T,
                                     leaf_side).T.reshape(nb, n_rhs, n_e)
    tm["p2m"] = time.perf_counter() - t0

    # M2M (engine.py:321-334), levels depth..1 -> depth-1..0.
    t0 = time.perf_counter()
    for lvl in range(depth, 0, -1):
        kids = st.level_keys(lvl)
        prow = np.searchsorted(st.level_keys(lvl - 1), parent_codes(kids))
        cidx = child_index_codes(kids)
        n_par = st.level_keys(lvl - 1).shape[0]
        stacked = np.zeros((n_par, 8, n_e, n_rhs), dtype=dtype)
        stacked[prow, cidx] = mult[lvl].transpose(0, 2, 1)
        stacked = stacked.transpose(1, 2, 0, 3).reshape(8 * n_e, n_par * n_rhs)
        out = np.empty((n_e, n_par * n_rhs), dtype=dtype)
        step = max(1, cfg.m2m_block) * n_rhs
        for c0 in range(0, n_par * n_rhs, step):
            c1 = min(c0 + step, n_par * n_rhs)
            out[:, c0:c1] = _solve(exp.up_inv, exp.m2m_kernels @ stacked[:, c0:c1], 1.0)
        mult[lvl - 1][:] = out.reshape(n_e, n_par, n_rhs).transpose(1, 2, 0)
    tm["m2m"] = time.perf_counter() - t0

    # Downward pass (engine.py:337-375).
    loc = [np.zeros((tt.level_keys(l).shape[0], n_rhs, n_e), dtype=dtype)
           for l in range(depth + 1)]
    tm["m2l"] = tm["l2l"] = 0.0
    for lvl in range(2, depth + 1):
        t0 = time.perf_counter()
        side = inst.domain.box_side(lvl)
        n_t = tt.level_keys(lvl).shape[0]
        if cfg.backend == "blas":
            check = apply_level(inst.blas_ops, inst.buckets[lvl], mult[lvl], n_t, 1.0 / side)
        else:
            check = m2l_fft_level(inst.fft_ops, inst.halo_plans[lvl], mult[lvl], 1.0 / side,
                                  workers=threads)
        loc[lvl] += _solve(exp.down_inv, check.reshape(n_t * n_rhs, n_c).T,
                           side).T.reshape(n_t, n_rhs, n_e)
        tm["m2l"] += time.perf_counter() - t0
        if lvl < depth:
            t0 = time.perf_counter()
            kids = tt.level_keys(lvl + 1)
            prow = np.searchsorted(tt.level_keys(lvl), parent_codes(kids))
            cidx = child_index_codes(kids)
            x = loc[lvl].reshape(n_t * n_rhs, n_e).T
            y = np.empty((8 * n_e, n_t * n_rhs), dtype=dtype)
            step = max(1, cfg.m2m_block) * n_rhs
            for c0 in range(0, n_t * n_rhs, step):
                c1 = min(c0 + step, n_t * n_rhs)
                w = c1 - c0
                ph = (exp.l2l_kernels @ x[:, c0:c1]).reshape(8, n_c, w)
                ph = ph.transpose(1, 0, 2).reshape(n_c, 8 * w)
                sol = _solve(exp.down_inv, ph, 0.5)
                y[:, c0:c1] = sol.reshape(n_e, 8, w).transpose(1, 0, 2).reshape(8 * n_e, w)
            y = y.reshape(8, n_e, n_t, n_rhs)
            loc[lvl + 1][:] += y[cidx, :, prow, :].transpose(0, 2, 1)
            tm["l2l"] += time.perf_counter() - t0

    # L2P (engine.py:377-389).
    t0 = time.perf_counter()
    pot = np.zeros((tt.n_points, n_rhs), dtype=dtype)
    equiv = np.ascontiguousarray(
        leaf_centers(tt)[:, None, :] + leaf_surface_base(cfg.order_equiv, leaf_side,
                                                         cfg.outer_scale)[None], dtype=dtype)
    for i in range(tt.leaves.shape[0]):
        s0 = int(tt.leaf_starts[i])
        s1 = s0 + int(tt.leaf_counts[i])
        g = equiv[i]
        k = laplace_matrix(tx[s0:s1], ty[s0:s1], tz[s0:s1], np.ascontiguousarray(g[:, 0]),
                           np.ascontiguousarray(g[:, 1]), np.ascontiguousarray(g[:, 2]), threads)
        pot[s0:s1] = k @ loc[depth][i].T
    tm["l2p"] = time.perf_counter() - t0

    # P2P (engine.py:391-397) on the reference's gathered layout.
    t0 = time.perf_counter()
    near_idx, near_off = inst.near.source_rows(st)
    leaf_of_target = np.repeat(np.arange(tt.leaves.shape[0], dtype=np.int64), tt.leaf_counts)
    p2p_blocked(tx, ty, tz, leaf_of_target, sx[near_idx], sy[near_idx], sz[near_idx],
                np.ascontiguousarray(q_tree[near_idx]), near_off, pot, threads)
    tm["p2p"] = time.perf_counter() - t0
    if state is not None:
        state["multipoles"] = mult
        state["locals"] = loc
    out = np.empty_like(pot)
    out[tt.perm] = pot
    return out


def gradient_matrix(t, s):
    """grad_t K(t, s) for K = 1/(4 pi |t - s|): (nt, ns, 3) float64, zero where
    t == s.  No reference counterpart (the reference is potential-only); the
    gradient of config 3 is checked against this and direct_gradient."""
    d = np.asarray(t, dtype=np.float64)[:, None, :] - np.asarray(s, dtype=np.float64)[None, :, :]
    r2 = np.einsum("ijk,ijk->ij", d, d)
    with np.errstate(divide="ignore"):
        w = np.where(r2 > 0, 1.0 / (4.0 * np.pi * r2 * np.sqrt(np.where(r2 > 0, r2, 1.0))), 0.0)
    return -d * w[:, :, None]


def direct_gradient(sources, charges, targets, chunk=2048):
    """Float64 direct-sum potential gradient at every target: (nt, n_rhs, 3)."""
    src = np.asarray(sources, dtype=np.float64).reshape(-1, 3)
    tgt = np.asarray(targets, dtype=np.float64).reshape(-1, 3)
    q = np.asarray(charges, dtype=np.float64).reshape(src.shape[0], -1)
    out = np.zeros((tgt.shape[0], q.shape[1], 3))
    for i0 in range(0, tgt.shape[0], chunk):
        g = gradient_matrix(tgt[i0:i0 + chunk], src)          # (c, ns, 3)
        out[i0:i0 + chunk] = np.einsum("isk,sr->irk", g, q)
    return out


def fmm_gradient(inst, charges, state):
    """The FMM gradient in float64 from the local expansions a previous
    ``evaluate(..., state=state)`` left in ``state["locals"]``: per target
    leaf, grad of the downward-equivalent-surface field (the L2P operator
    differentiated) plus the near-field direct gradient over the reference's
    P2P source rows (engine.py:224-256).  Caller order, (nt, n_rhs, 3)."""
    from paper_2408_07436_b200.engine import as_charge_matrix, leaf_centers, leaf_surface_base
    cfg = inst.config
    st, tt = inst.source_tree, inst.target_tree
    depth = cfg.depth
    q = as_charge_matrix(np.asarray(charges), st.n_points)
    q_tree = np.asarray(q, dtype=np.float64)[st.perm]
    loc = np.asarray(state["locals"][depth], dtype=np.float64)        # (n_leaves, n_rhs, n_e)
    equiv = leaf_centers(tt)[:, None, :] + leaf_surface_base(
        cfg.order_equiv, inst.domain.box_side(depth), cfg.outer_scale)[None]
    near_idx, near_off = inst.near.source_rows(st)
    tpts = np.stack([tt.x, tt.y, tt.z], axis=1)
    spts = np.stack([st.x, st.y, st.z], axis=1)
    grad = np.zeros((tt.n_points, q.shape[1], 3))
    for i in range(tt.leaves.shape[0]):
        s0 = int(tt.leaf_starts[i])
        s1 = s0 + int(tt.leaf_counts[i])
        t = tpts[s0:s1]
        grad[s0:s1] += np.einsum("tsk,rs->trk", gradient_matrix(t, equiv[i]), loc[i])
        rows = near_idx[near_off[i]:near_off[i + 1]]
        grad[s0:s1] += np.einsum("tsk,sr->trk", gradient_matrix(t, spts[rows]), q_tree[rows])
    out = np.empty_like(grad)
    out[tt.perm] = grad
    return out


def direct(sources, charges, targets, dtype=np.float64, threads=None):
    """kernel.direct_potentials (kernel.py:83-103): the O(N^2) oracle."""
    src = np.asarray(sources, dtype=np.float64).reshape(-1, 3)
    tgt = np.asarray(targets, dtype=np.float64).reshape(-1, 3)
    q = np.asarray(charges, dtype=dtype).reshape(src.shape[0], -1)
    out = np.zeros((tgt.shape[0], q.shape[1]), dtype=dtype)
    laplace_potentials(*(np.ascontiguousarray(tgt[:, a], dtype=dtype) for a in range(3)),
                       *(np.ascontiguousarray(src[:, a], dtype=dtype) for a in range(3)),
                       np.ascontiguousarray(q), out, threads)
    return out
