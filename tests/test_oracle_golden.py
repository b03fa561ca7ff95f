"""Pin the oracle restatement against the reference's own outputs (golden
vectors produced by tests/golden/make_golden.py from the unmodified
reference).  CPU only."""

import numpy as np
import pytest

from conftest import golden
from oracle import port
from paper_2408_07436_b200 import FmmConfig, setup


@pytest.mark.parametrize("tag", ["float32", "float64"])
def test_hot_loops(tag):
    g = golden("hotloops")
    a = lambda k: g[f"{tag}_{k}"]                     # noqa: E731
    pot = np.zeros_like(a("pot"))
    port.laplace_potentials(a("tx"), a("ty"), a("tz"), a("sx"), a("sy"), a("sz"), a("q"), pot)
    assert np.array_equal(pot, a("pot")) or np.allclose(pot, a("pot"), rtol=1e-6 if tag == "float32" else 1e-14)
    mat = port.laplace_matrix(a("tx"), a("ty"), a("tz"), a("sx"), a("sy"), a("sz"))
    assert np.array_equal(mat, a("mat"))
    out = np.full_like(a("p2p_out"), 0.5)
    port.p2p_blocked(a("p2p_tx"), a("p2p_ty"), a("p2p_tz"), a("p2p_lot"), a("p2p_sx"),
                     a("p2p_sy"), a("p2p_sz"), a("p2p_q"), a("p2p_off"), out)
    assert np.allclose(out, a("p2p_out"), rtol=1e-6 if tag == "float32" else 1e-14, atol=0)


@pytest.mark.parametrize("tag", ["complex64", "complex128"])
def test_hadamard(tag):
    g = golden("hotloops")
    phat = np.full_like(g[f"{tag}_phat"], 0.25)
    port.hadamard_m2l(g[f"{tag}_khat"], g[f"{tag}_qhat"], g[f"{tag}_halo"], phat)
    want = g[f"{tag}_phat"]
    assert np.abs(phat - want).max() <= (1e-6 if tag == "complex64" else 1e-13) * np.abs(want).max()


@pytest.mark.parametrize("name", ["c1", "blas_f32", "fft_f64", "fft_f32", "blas_f64_pc",
                                  "blas_f64_rhs"])
def test_evaluate(name):
    g = golden("eval_" + name)
    kw = {k[4:]: g[k].item() for k in g.files if k.startswith("cfg_")}
    inst = setup(g["points"], g["points"], FmmConfig(**kw))
    got = port.evaluate(inst, g["charges"])
    want = g["potentials"].reshape(got.shape)
    # same host as the generator -> bit-identical; elsewhere BLAS rounding may differ
    tol = 1e-6 if want.dtype == np.float32 else 1e-13
    assert np.abs(got - want).max() <= tol * np.abs(want).max()


def test_gradient_restatement_against_direct_sum():
    """The oracle's FMM gradient (no reference counterpart) converges to the
    float64 direct-sum gradient at the accuracy of the expansion order."""
    from oracle import port
    from paper_2408_07436_b200 import FmmConfig, setup
    pts = np.random.default_rng(7).random((2000, 3))
    q = np.random.default_rng(11).uniform(-1, 1, 2000)
    exact = port.direct_gradient(pts, q, pts)
    errs = []
    for p in (4, 6):
        inst = setup(pts, pts, FmmConfig(depth=3, order_equiv=p, backend="fft", precision="f64"))
        st = {}
        port.evaluate(inst, q, state=st)
        g = port.fmm_gradient(inst, q, st)
        errs.append(np.linalg.norm(g - exact) / np.linalg.norm(exact))
    assert errs[0] < 1e-3 and errs[1] < errs[0] / 10
    # finite-difference check of the direct gradient itself (off-source points)
    h = 1e-5
    t = np.random.default_rng(5).random((5, 3))
    g = port.direct_gradient(pts, q, t)
    for k in range(3):
        e = np.zeros(3)
        e[k] = h
        fd = (port.direct(pts, q, t + e) - port.direct(pts, q, t - e)) / (2 * h)
        assert np.allclose(fd[:, 0], g[:, 0, k], rtol=1e-5, atol=1e-8 * np.abs(g).max())
