"""The reference arm's instance builder reproduces the reference's own setup
exactly (CPU; needs the compiled reference in oracle/_ref)."""

import numpy as np
import pytest

from oracle import reference_available

pytestmark = pytest.mark.skipif(not reference_available(),
                                reason="oracle/_ref not built (python oracle/build_ref.py)")


def test_bridge_matches_reference_setup():
    from oracle import import_reference
    from oracle.ref_bridge import make_reference_instance
    kifmm3d = import_reference()
    from kifmm3d import engine
    pts = np.random.default_rng(7).random((3000, 3))
    tgt = np.random.default_rng(8).random((2000, 3))
    kw = dict(depth=3, order_equiv=4, backend="blas", precision="f32", sigma_min=1e-6)
    a = engine.setup(pts, tgt, engine.FmmConfig(**kw))
    b = make_reference_instance(pts, tgt, **kw)
    for name in ("_near_idx", "_near_offsets", "_near_sx", "_near_sy", "_near_sz",
                 "_leaf_of_target", "_sx", "_tx", "_src_check", "_tgt_equiv"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name
    assert a.n_near_pairs == b.n_near_pairs
    q = np.random.default_rng(11).random(3000)
    assert np.array_equal(a.evaluate(q), b.evaluate(q))
