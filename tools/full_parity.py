"""Per-target parity against the UNMODIFIED reference at the full BASELINE
sizes (configs 2-5), run on the GPU box (the reference's SVD-truncated
operators depend on the host LAPACK, so both sides must run on one host).

    python tools/full_parity.py all            # every case, one subprocess each
    python tools/full_parity.py c3             # one case

For each case: the same seeded inputs (points seed 7, charges
seed 11) go through
  * ours: ``setup`` + ``FmmInstance.evaluate`` (GPU), ``relative_error``;
  * the reference: oracle/_ref (Cython-compiled /root/reference, via
    oracle/ref_bridge.py) ``evaluate`` on all host cores,
    ``relative_error`` (engine.py:270-404, 412-451);
and the record holds the strict per-target failure count at the north_star
tolerance (1e-5 f32 / 1e-10 f64), max / median per-target relative
difference, the normwise ratio ||d||_inf / ||phi||_inf, the floored ratio
|d| / max(|phi|, 1e-3 ||phi||_inf) with its failure count, both
``relative_error`` values, and both sides' error against an f64 direct sum
on 4096 sampled targets.  Records go to profiles/r2/parity_full/<case>.json;
tests/test_full_parity_records.py asserts them.

ORACLE use: this is test infrastructure (it imports oracle/), not product.
"""

from __future__ import annotations

import json
import os
import platform
import subprocess
import sys
import time

_n = str(os.cpu_count() or 1)
for _k, _v in (("OMP_WAIT_POLICY", "PASSIVE"), ("OMP_NUM_THREADS", _n), ("KIFMM_THREADS", _n)):
    os.environ.setdefault(_k, _v)

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "profiles", "r2", "parity_full")


def uniform(n, signed=False):
    pts = np.random.default_rng(7).random((n, 3))                   # generate_points("uniform-cube")
    rng = np.random.default_rng(11)
    return pts, (rng.uniform(-1, 1, n) if signed else rng.random(n))


def sphere(n):
    v = np.random.default_rng(7).standard_normal((n, 3))             # generate_points("sphere-surface")
    pts = (v / np.linalg.norm(v, axis=1)[:, None] + 1.0) / 2.0       # scaled into [0,1]^3
    return pts, np.random.default_rng(11).standard_normal(n)


C4 = dict(depth=6, order_equiv=6, sigma_min=1e-6)
CASES = {
    "c2": (lambda: uniform(1_000_000),
           dict(depth=5, order_equiv=4, backend="blas", precision="f32", sigma_min=1e-6)),
    "c3": (lambda: uniform(1_000_000, signed=True),
           dict(depth=5, order_equiv=8, backend="fft", precision="f64")),
    "c4_blas_f32": (lambda: uniform(8_000_000), dict(C4, backend="blas", precision="f32")),
    "c4_blas_f64": (lambda: uniform(8_000_000), dict(C4, backend="blas", precision="f64")),
    "c4_fft_f32": (lambda: uniform(8_000_000), dict(C4, backend="fft", precision="f32")),
    "c4_fft_f64": (lambda: uniform(8_000_000), dict(C4, backend="fft", precision="f64")),
    "c5": (lambda: sphere(4_000_000),
           dict(depth=7, order_equiv=10, backend="blas", precision="f64", sigma_min=1e-12)),
}
TOL = {"f32": 1e-5, "f64": 1e-10}


def direct_sample(pts, q, idx):
    """f64 direct sum at the sampled targets (GPU, kernel-level boundary)."""
    from paper_2408_07436_b200 import hotloops
    c = lambda a, k: np.ascontiguousarray(a[:, k])                   # noqa: E731
    t = pts[idx]
    out = np.zeros((idx.shape[0], 1))
    hotloops.laplace_potentials(c(t, 0), c(t, 1), c(t, 2), c(pts, 0), c(pts, 1), c(pts, 2),
                                np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 1), out)
    return out[:, 0]


def err_stats(phi, ref):
    rel = np.abs(phi - ref) / np.abs(ref)
    return dict(mean=float(rel.mean()), max=float(rel.max()),
                normwise=float(np.abs(phi - ref).max() / np.abs(ref).max()))


def run_case(name):
    import torch
    from paper_2408_07436_b200 import FmmConfig, setup
    make, kw = CASES[name]
    pts, q = make()
    rec = dict(case=name, n_points=int(pts.shape[0]), config=kw,
               seeds={"points": 7, "charges": 11}, host=dict(
                   cpu_count=os.cpu_count(), cpu=_cpu_model() or platform.processor(),
                   gpu=torch.cuda.get_device_name(0) if torch.cuda.is_available() else None))
    # ---- ours (GPU)
    t0 = time.perf_counter()
    inst = setup(pts, pts, FmmConfig(**kw))
    rec["ours_setup_s"] = time.perf_counter() - t0
    got = inst.evaluate(q)
    t0 = time.perf_counter()
    got = inst.evaluate(q)
    rec["ours_evaluate_s"] = time.perf_counter() - t0
    rec["ours_relative_error"] = list(inst.relative_error(got))
    if kw["backend"] == "blas":
        bd = inst.device.blas
        rec["ours_sweep"] = ("tcgen05 3xTF32 (tensor memory)" if getattr(bd, "tmem", False) else
                             "tcgen05 3xTF32 (TMA)" if bd.tc else
                             "DMMA factored (compress + expand)" if getattr(bd, "factored", False)
                             else "DMMA dense cores")
    idx = np.sort(np.random.default_rng(5).choice(pts.shape[0], 4096, replace=False))
    direct = direct_sample(pts, q, idx)
    rec["ours_vs_direct_4096"] = err_stats(np.asarray(got, np.float64)[idx], direct)
    del inst
    torch.cuda.empty_cache()
    # ---- reference (CPU, this host)
    from oracle.ref_bridge import make_reference_instance
    t0 = time.perf_counter()
    ref = make_reference_instance(pts, pts, threads=os.cpu_count(), **kw)
    rec["reference_setup_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    want = np.asarray(ref.evaluate(q))
    rec["reference_evaluate_s"] = time.perf_counter() - t0
    rec["reference_timings"] = {k: float(v) for k, v in ref.timings.items()}
    rec["reference_relative_error"] = list(ref.relative_error(want))
    rec["reference_vs_direct_4096"] = err_stats(np.asarray(want, np.float64)[idx], direct)
    # the reference against itself: single-threaded OpenBLAS changes only
    # BLAS rounding (bounds how closely any implementation can match it)
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1, user_api="blas"):
        want1 = np.asarray(ref.evaluate(q), np.float64)
    w0 = np.asarray(want, np.float64)
    d1 = np.abs(want1 - w0)
    sc = np.abs(w0).max()
    rec["reference_vs_itself"] = dict(
        max_rel=float((d1 / np.abs(w0)).max()), normwise=float(d1.max() / sc),
        floored_max=float((d1 / np.maximum(np.abs(w0), 1e-3 * sc)).max()),
        strict_failures=int((d1 / np.abs(w0) > TOL[kw["precision"]]).sum()),
        note="the reference evaluated again with single-threaded OpenBLAS")
    # ---- per-target comparison
    g = np.asarray(got, np.float64)
    w = np.asarray(want, np.float64)
    assert g.shape == w.shape, (g.shape, w.shape)
    d = np.abs(g - w)
    rel = d / np.abs(w)
    scale = np.abs(w).max()
    floored = d / np.maximum(np.abs(w), 1e-3 * scale)
    tol = TOL[kw["precision"]]
    rec["parity"] = dict(
        tol=tol, n_targets=int(w.size), max_rel=float(rel.max()), median_rel=float(np.median(rel)),
        p99999_rel=float(np.quantile(rel, 0.99999)),
        strict_failures=int((rel > tol).sum()), normwise=float(d.max() / scale),
        floored_max=float(floored.max()), floored_failures=int((floored > tol).sum()),
        relative_error_gap=abs(rec["ours_relative_error"][0] - rec["reference_relative_error"][0]),
        signed_charges=bool((q < 0).any()))
    rec["dtype_ours"] = str(np.asarray(got).dtype)
    rec["dtype_reference"] = str(np.asarray(want).dtype)
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"{name}.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps(dict(case=name, **rec["parity"])), flush=True)


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def main(argv):
    which = argv[1] if len(argv) > 1 else "all"
    if which != "all":
        run_case(which)
        return 0
    rc = 0
    for name in (argv[2].split(",") if len(argv) > 2 else CASES):
        r = subprocess.run([sys.executable, os.path.abspath(__file__), name])
        rc |= r.returncode
    return rc


if __name__ == "__main__":
    sys.exit(main(sys.argv))
