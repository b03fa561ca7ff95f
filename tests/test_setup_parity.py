"""Host setup (trees, operators, per-level plans) reproduces the reference's
setup on the same inputs (golden vectors from the reference itself)."""

import hashlib

import numpy as np
import pytest

from conftest import golden, uniform_points
from paper_2408_07436_b200 import FmmConfig, setup
from paper_2408_07436_b200.engine import ConfigError

NAMES = ["c1", "blas_f32", "fft_f64", "fft_f32", "blas_f64_pc", "blas_f64_rhs"]


def _cfg(g):
    kw = {k[4:]: g[k].item() for k in g.files if k.startswith("cfg_")}
    return FmmConfig(**kw)


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.int64).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module", params=NAMES)
def case(request):
    g = golden("eval_" + request.param)
    inst = setup(g["points"], g["points"], _cfg(g))
    return request.param, g, inst


def test_operators_match_reference(case):
    name, g, inst = case
    if inst.config.backend == "blas":
        ops = inst.blas_ops
        # same machine -> bit-identical; other hosts may differ in LAPACK rounding
        assert np.allclose(ops.u, g["u"], rtol=0, atol=1e-12 if ops.u.dtype == np.float64 else 1e-5)
        assert np.allclose(ops.s, g["s"], rtol=0, atol=1e-12 if ops.s.dtype == np.float64 else 1e-5)
        assert np.array_equal(ops.ranks, g["ranks"])
    else:
        kh = inst.fft_ops.khat
        tol = 1e-12 if kh.dtype == np.complex128 else 1e-5
        for key, sl in (("khat_f0", kh[0]), ("khat_fl", kh[-1])):
            want = g[key]
            assert np.abs(sl - want).max() <= tol * np.abs(want).max()
        assert np.isclose(np.abs(kh).sum(), float(g["khat_abs_sum"]), rtol=1e-6)


def test_near_field_plan_matches_reference(case):
    name, g, inst = case
    rows, offs = inst.near.source_rows(inst.source_tree)
    assert _digest(rows, offs) == str(g["near_sha"])


def test_bucket_plan_covers_every_pair(case):
    name, g, inst = case
    if inst.config.backend != "blas":
        pytest.skip("blas only")
    for lvl, plan in inst.blas_plans.items():
        b = inst.buckets[lvl]
        assert plan.n_pairs == sum(p[0].shape[0] for p in b.pairs if p is not None)
        assert int((plan.src >= 0).sum()) == plan.n_pairs
        valid = plan.tile_targets >= 0
        assert np.array_equal(np.sort(plan.tile_targets[valid]),
                              np.arange(inst.target_tree.level_keys(lvl).shape[0]))


def test_hadamard_tiles_reproduce_halo(case):
    """The tiled Hadamard's plan (csrc/hadamard.cu) addresses exactly the
    halo table's sources, with the bank invariants the kernel relies on:
    column 32w + 4g + j holds a target of parity class g, a source sits in a
    slot of its own class, and absent sources map to zero row UMAX + class."""
    from paper_2408_07436_b200.m2l_fft import (HAD_OFFSET_PARITY, HAD_TILE, HAD_UMAX,
                                               plan_hadamard_tiles)
    name, g, inst = case
    if inst.config.backend != "fft":
        pytest.skip("fft only")
    col_class = (np.arange(HAD_TILE) >> 2) & 7
    for lvl, hp in inst.halo_plans.items():
        for umax in (HAD_UMAX, 64):                    # 64 forces tile splitting
            t = plan_hadamard_tiles(hp.halo, hp.src_color, hp.tgt_color, umax=umax)
            assert t.begin[0] == 0 and t.begin[-1] == hp.halo.shape[0]
            for k in range(t.n_tiles):
                b, e = t.begin[k], t.begin[k + 1]
                assert 0 < e - b <= HAD_TILE
                table = t.src[t.src_off[k]:t.src_off[k + 1]]
                assert table.shape[0] <= umax or e - b == 1
                used = table >= 0
                assert np.array_equal(hp.src_color[table[used]], np.flatnonzero(used) % 8)
                tcol = t.tcol[k].astype(np.int64)
                filled = tcol >= 0
                assert np.array_equal(np.sort(tcol[filled]), np.arange(e - b))
                assert np.array_equal(hp.tgt_color[b + tcol[filled]], col_class[filled])
                sl = t.slots[k].astype(np.int64)              # (26, HAD_TILE)
                want_class = col_class[None, :] ^ HAD_OFFSET_PARITY[:, None]
                assert np.array_equal(sl % 8, want_class)
                absent = sl >= umax
                assert np.array_equal(sl[absent], umax + want_class[absent])
                got = np.where(absent, -1, table[np.minimum(sl, table.shape[0] - 1)])
                assert np.array_equal(got[:, filled].T, hp.halo[b + tcol[filled]])


def test_sparse_tile_lists_match_the_source_table(case):
    """Host logic of the sparse float64 sweep: vector lists and 8-row-group
    masks reproduce exactly where the BLAS plan's source table is populated."""
    from paper_2408_07436_b200.device import sparse_tile_lists
    name, g, inst = case
    if inst.config.backend != "blas":
        pytest.skip("blas only")
    for lvl, plan in inst.blas_plans.items():
        nt = plan.tile_class.shape[0]
        gmask, jlist, jcount = sparse_tile_lists(plan.src, nt)
        pres = (plan.src.reshape(nt, 16, 8, 189) >= 0).any(axis=2)
        for t in range(nt):
            bits = np.array([[(int(gmask[t, j]) >> k) & 1 for k in range(16)] for j in range(189)])
            assert np.array_equal(bits.T.astype(bool), pres[t])
            want = np.flatnonzero(pres[t].any(axis=0))
            assert jcount[t] == want.shape[0]
            assert np.array_equal(jlist[t, : jcount[t]], want)
            assert (jlist[t, jcount[t]:] == -1).all()


def test_config_validation_mirrors_reference():
    for bad in (dict(depth=1), dict(order_equiv=1), dict(order_equiv=6, order_check=5),
                dict(backend="magic"), dict(backend="fft", order_equiv=6, order_check=8),
                dict(precision="f16"), dict(sigma_min=-1.0), dict(alpha=-0.5),
                dict(oversamples=0), dict(block_size=0), dict(n_rhs=0),
                dict(m2l_strategy="surprise"), dict(inner_scale=3.0, outer_scale=2.0)):
        with pytest.raises(ConfigError):
            FmmConfig(**bad)
    assert FmmConfig(precision="f32").dtype == np.float32
    assert FmmConfig(threads=64).resolved_m2l_strategy() == "bucket-threads"


def test_setup_rejects_empty_clouds():
    pts = uniform_points(10)
    with pytest.raises(ConfigError):
        setup(np.empty((0, 3)), pts, FmmConfig(depth=2, order_equiv=3))
    with pytest.raises(ConfigError):
        setup(pts, np.empty((0, 3)), FmmConfig(depth=2, order_equiv=3))


def test_locality_vector_order_is_a_permutation():
    """The tensor-memory sweep's class vector order (device.py
    locality_transfer_table) lists exactly each class's 189 admissible
    vectors, grouped by source sub-lattice."""
    from paper_2408_07436_b200.device import locality_transfer_table
    from paper_2408_07436_b200.octree import class_transfer_table, transfer_offsets
    loc, base = locality_transfer_table(), class_transfer_table()
    offs = transfer_offsets()
    for cls in range(8):
        assert sorted(loc[cls].tolist()) == sorted(base[cls].tolist())
        par = np.array([(cls >> 2) & 1, (cls >> 1) & 1, cls & 1])
        q = par[None, :] + offs[loc[cls]]
        sp = ((q[:, 0] & 1) << 2) | ((q[:, 1] & 1) << 1) | (q[:, 2] & 1)
        assert np.all(np.diff(sp) >= 0)


def test_tmem_core_packing_layout():
    """pack_tmem_cores: per vector [B_hi | B_lo], each K-major [n/8][k/4][n%8][k%4]."""
    from paper_2408_07436_b200.device import pack_tmem_cores
    rng = np.random.default_rng(0)
    kp = 16
    hi = rng.random((3, 13, 13)).astype(np.float32)
    lo = rng.random((3, 13, 13)).astype(np.float32)
    out = pack_tmem_cores(hi, lo, kp)
    assert out.shape == (3, 2 * kp * kp)
    for t in range(3):
        for half, src in ((0, hi), (1, lo)):
            blk = out[t, half * kp * kp:(half + 1) * kp * kp].reshape(kp // 8, kp // 4, 8, 4)
            dense = blk.transpose(0, 2, 1, 3).reshape(kp, kp)
            assert np.array_equal(dense[:13, :13], src[t])
            assert not dense[13:].any() and not dense[:, 13:].any()


def test_factored_sweep_widths():
    """Width classes of the factored float64 sweep (device.factored_widths):
    ktp = 16 * ntw * slabs covers the rank with at most 10 fragments per slab
    (csrc/m2l_factored.cu dispatches ntw = 1..10); rank 0 stays 0."""
    from paper_2408_07436_b200.device import factored_widths
    ranks = np.array([0, 1, 16, 17, 54, 160, 161, 198, 320, 321, 483])
    ktp, ntw, slabs = factored_widths(ranks)
    assert ktp[0] == 0 and ntw[0] == 0
    live = ranks > 0
    assert np.all(ktp[live] >= ranks[live]) and np.all(ktp % 16 == 0)
    assert np.all(ktp[live] == 16 * ntw[live] * slabs[live])
    assert np.all((ntw[live] >= 1) & (ntw[live] <= 10))
    # no more padding than one 16-column step per slab
    assert np.all(ktp[live] - ranks[live] < 16 * slabs[live] + 16)
    assert list(ktp[[2, 3, 5, 6, 7]]) == [16, 32, 160, 192, 224]
