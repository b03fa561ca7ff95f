"""ORACLE - baseline infrastructure only (bench.py's reference arm and
cpu_baseline leg, tests).

Builds an ``FmmInstance`` of the UNMODIFIED reference package (the
Cython-compiled copy in oracle/_ref) for large inputs.  Every field is
produced by the reference's own functions (``Octree``,
``ExpansionOperators``, ``m2l_blas.precompute``/``bucket_level``,
``m2l_fft.precompute_fft_operators``/``build_halo_plan``, the per-leaf
surfaces and parent maps of ``engine.setup``), except the near-field gather
plan: the reference builds it with a per-leaf Python loop (engine.py:224-256)
that takes ~6 min at 1M points and ~1 h at 8M.  We fill those arrays from
an equivalent vectorised construction instead;
tests/test_ref_bridge.py asserts the result is identical to the reference's
own ``setup`` (bit-for-bit, all fields) on small inputs.  ``evaluate`` - the
timed path - is the reference's, untouched.
"""

from __future__ import annotations

import time

import numpy as np

from . import import_reference


def make_reference_instance(sources, targets, **config_kwargs):
    kifmm3d = import_reference()
    from kifmm3d import engine as E
    from kifmm3d import m2l_blas, m2l_fft
    from kifmm3d.expansion import ExpansionOperators
    from kifmm3d.octree import Domain, Octree, child_index_codes, parent_codes

    t0 = time.perf_counter()
    config = E.FmmConfig(**config_kwargs)
    src = np.ascontiguousarray(np.asarray(sources, dtype=np.float64).reshape(-1, 3))
    tgt = np.ascontiguousarray(np.asarray(targets, dtype=np.float64).reshape(-1, 3))
    domain = Domain.from_points(np.vstack([src, tgt]))
    st = Octree(src, config.depth, domain)
    tt = Octree(tgt, config.depth, domain)
    dtype = config.dtype
    exp = ExpansionOperators(config.order_equiv, config.resolved_order_check(), dtype=dtype,
                             alpha=config.alpha, cutoff=config.svd_cutoff,
                             inner_scale=config.inner_scale, outer_scale=config.outer_scale)
    inst = E.FmmInstance(config=config, domain=domain, source_tree=st, target_tree=tt,
                         expansions=exp)
    if config.backend == "blas":
        inst.blas_ops = m2l_blas.precompute(
            config.order_equiv, config.resolved_order_check(), sigma_min=config.sigma_min,
            rank_estimate=config.rank_estimate, oversamples=config.oversamples, seed=config.seed,
            dtype=dtype, inner_scale=config.inner_scale,
            level_scale=1.0 / domain.box_side(config.depth))
        for lvl in range(2, config.depth + 1):
            inst.buckets[lvl] = m2l_blas.bucket_level(st, tt, lvl)
    else:
        inst.fft_ops = m2l_fft.precompute_fft_operators(
            config.order_equiv, dtype=dtype, inner_scale=config.inner_scale,
            workers=config.threads)
        for lvl in range(2, config.depth + 1):
            inst.halo_plans[lvl] = m2l_fft.build_halo_plan(st, tt, lvl)
    inst._sx = np.ascontiguousarray(st.x, dtype=dtype)
    inst._sy = np.ascontiguousarray(st.y, dtype=dtype)
    inst._sz = np.ascontiguousarray(st.z, dtype=dtype)
    inst._tx = np.ascontiguousarray(tt.x, dtype=dtype)
    inst._ty = np.ascontiguousarray(tt.y, dtype=dtype)
    inst._tz = np.ascontiguousarray(tt.z, dtype=dtype)
    inst._src_check = E._leaf_surfaces(st, config.resolved_order_check(), config.outer_scale,
                                       dtype)
    inst._tgt_equiv = E._leaf_surfaces(tt, config.order_equiv, config.outer_scale, dtype)
    inst._up_maps, inst._down_maps = {}, {}
    for lvl in range(1, config.depth + 1):
        for tree, maps in ((st, inst._up_maps), (tt, inst._down_maps)):
            kids = tree.level_keys(lvl)
            prow = np.searchsorted(tree.level_keys(lvl - 1), parent_codes(kids))
            maps[lvl] = (prow.astype(np.int64), child_index_codes(kids))
    # near field: vectorised equivalent of engine.py:224-256
    from paper_2408_07436_b200.engine import near_field_plan
    from paper_2408_07436_b200.octree import Octree as OurOctree
    ours_s = OurOctree(src, config.depth, _our_domain(domain))
    ours_t = OurOctree(tgt, config.depth, _our_domain(domain))
    plan = near_field_plan(ours_s, ours_t)
    inst._near_idx, inst._near_offsets = plan.source_rows(ours_s)
    inst._near_sx = inst._sx[inst._near_idx]
    inst._near_sy = inst._sy[inst._near_idx]
    inst._near_sz = inst._sz[inst._near_idx]
    inst._leaf_of_target = np.repeat(np.arange(tt.leaves.shape[0], dtype=np.int64),
                                     tt.leaf_counts)
    counts = np.diff(inst._near_offsets)
    inst.n_near_pairs = int((counts * tt.leaf_counts).sum())
    inst.setup_seconds = time.perf_counter() - t0
    return inst


def _our_domain(d):
    from paper_2408_07436_b200.octree import Domain
    return Domain(tuple(d.origin), d.side)
