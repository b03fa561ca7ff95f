"""Small evaluates that launch every kernel family once or twice, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck, one tool per
run):  compute-sanitizer --tool racecheck python tools/sanitize_small.py

Covers: device tree build, f32 BLAS (tensor-memory sweep, fused P2M, mutual
near field, L2P from the folded solve, chains, GEMMs), f32 BLAS at p = 6 (the
TMA sweep, k > 64), f64 BLAS (DMMA sweep, DMMA GEMM), f64 FFT (forward and
inverse DFT, DMMA Hadamard) with the gradient pass, the level drop-ins
(cp.async tcgen05 sweep) and the kernel-level boundary (P2P CSR, Hadamard
gather)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2408_07436_b200 import FmmConfig, hotloops, m2l_blas, m2l_fft, setup
    torch.cuda.set_device(0)
    rng = np.random.default_rng(3)
    pts = rng.random((6000, 3))
    q = rng.random(6000)
    cases = [dict(depth=3, order_equiv=4, backend="blas", precision="f32", sigma_min=1e-6),
             dict(depth=3, order_equiv=6, backend="blas", precision="f32", sigma_min=1e-6),
             dict(depth=3, order_equiv=5, backend="blas", precision="f64", sigma_min=1e-12),
             dict(depth=3, order_equiv=4, backend="fft", precision="f64")]
    for kw in cases:
        inst = setup(pts, pts, FmmConfig(**kw))
        phi = inst.evaluate(q)
        assert np.all(np.isfinite(phi)), kw
        inst.evaluate(np.stack([q, 2 * q], axis=1))
        if kw["backend"] == "fft":
            inst.evaluate(q, gradient=True)
            lvl = 3
            m2l_fft.m2l_fft_level(inst.fft_ops, inst.halo_plans[lvl],
                                  rng.random((inst.source_tree.level_keys(lvl).shape[0], 1,
                                              inst.expansions.n_equiv)), 1.0)
        else:
            lvl = 3
            n_t = inst.target_tree.level_keys(lvl).shape[0]
            mult = rng.random((inst.source_tree.level_keys(lvl).shape[0], 1,
                               inst.expansions.n_equiv)).astype(inst.config.dtype)
            m2l_blas.apply_level(inst.blas_ops, inst.buckets[lvl], mult, n_t, 1.0)
        print("ok", kw, flush=True)
    # kernel-level boundary
    t = rng.random((3, 50))
    s_ = rng.random((3, 70))
    out = np.zeros((50, 1))
    hotloops.laplace_potentials(*t, *s_, rng.random((70, 1)), out)
    torch.cuda.synchronize()
    print("sanitize_small done")


if __name__ == "__main__":
    main()
