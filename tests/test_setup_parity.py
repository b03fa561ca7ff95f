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
