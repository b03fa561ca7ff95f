"""Device tree and plan build.

The reference builds its octrees and plans on the host (``octree.py:274-329``,
``engine.py:224-256``, ``m2l_blas.py:232-258``); the host restatement here
(``octree.Octree``, ``engine.near_field_plan``, ``m2l_blas.bucket_level`` +
``level_plan_from_buckets``) is vectorised numpy.  This module builds the same
objects on the GPU through the C ABI (``csrc/plan.cu``): Morton encode,
stable radix sort, run-length encode of the leaves, every coarser level by
parent-code uniquing, the near-field candidate table, and the target-
stationary BLAS-M2L source table.  Results are bit-identical to the host
build (tests/test_gpu_parity.py::test_device_setup_matches_host); the device
BLAS source table is kept on the device for the sweep.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .device import P, require_cuda, stream_handle, to_dev
from .octree import LEVEL_BITS, DomainError, Octree, class_transfer_table, transfer_offsets


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


def _u64(n):
    return torch.empty(max(int(n), 1), dtype=torch.int64, device=_dev())


def _temp(op, n, end_bit=64):
    out = np.zeros(1, dtype=np.int64)
    nat.call("kifmm_tree_temp_bytes", op, int(n), int(end_bit), out.ctypes.data)
    return torch.empty(max(int(out[0]), 1), dtype=torch.uint8, device=_dev()), int(out[0])


def _scalar(t):
    return int(t[:1].cpu().numpy()[0])


def octree(points, depth: int, domain) -> Octree:
    """Same tree as ``Octree(points, depth, domain)``, built on the device."""
    require_cuda()
    p = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3))
    n = p.shape[0]
    if n < 1:
        raise ValueError("a tree needs at least one point")
    s = stream_handle()
    pts = to_dev(p)
    codes = _u64(n)
    bad = torch.zeros(1, dtype=torch.int32, device=_dev())
    o = domain.origin
    nat.call("kifmm_tree_encode", P(pts), n, float(o[0]), float(o[1]), float(o[2]),
             float(domain.side), depth, P(codes), P(bad), s)
    if _scalar(bad):
        raise DomainError("a point lies outside the domain")
    end_bit = LEVEL_BITS + 3 * depth
    sorted_codes, perm = _u64(n), _u64(n)
    tmp, nb = _temp(0, n, end_bit)
    nat.call("kifmm_tree_sort", P(codes), n, end_bit, P(sorted_codes), P(perm), P(tmp), nb, s)
    leaves, counts, nrun = _u64(n), _u64(n), _u64(1)
    tmp, nb = _temp(1, n)
    nat.call("kifmm_tree_rle", P(sorted_codes), n, P(leaves), P(counts), P(nrun), P(tmp), nb, s)
    n_leaves = _scalar(nrun)
    levels = [None] * (depth + 1)
    levels[depth] = leaves[:n_leaves]
    scratch, nout = _u64(n_leaves), _u64(1)
    for lvl in range(depth - 1, -1, -1):
        child = levels[lvl + 1]
        par = _u64(child.shape[0])
        tmp, nb = _temp(2, child.shape[0])
        nat.call("kifmm_tree_parents", P(child), child.shape[0], P(scratch), P(par), P(nout),
                 P(tmp), nb, s)
        levels[lvl] = par[:_scalar(nout)]
    perm_h = perm.cpu().numpy()
    cnt = counts[:n_leaves].cpu().numpy()
    starts = np.concatenate([[0], np.cumsum(cnt)[:-1]]).astype(np.int64)
    lv = [l.cpu().numpy().view(np.uint64).copy() for l in levels]
    tree = Octree.from_arrays(depth, domain, perm_h, p[perm_h], starts, cnt.astype(np.int64), lv)
    tree.device_levels = levels                       # device copies (int64 storage of u64)
    return tree


def _dev_levels(tree):
    lv = getattr(tree, "device_levels", None)
    if lv is None:
        lv = [to_dev(k.view(np.int64)) for k in tree.levels]
        tree.device_levels = lv
    return lv


def near_field_plan(source_tree, target_tree):
    """Same plan as ``engine.near_field_plan``, candidates looked up on the device."""
    from .engine import NearFieldPlan
    require_cuda()
    depth = target_tree.depth
    tl = _dev_levels(target_tree)[depth]
    sl = _dev_levels(source_tree)[depth]
    ntl = target_tree.leaves.shape[0]
    rows_d = torch.empty(max(ntl, 1) * 27, dtype=torch.int64, device=_dev())
    nat.call("kifmm_near_field_rows", P(tl), ntl, depth, P(sl), source_tree.leaves.shape[0],
             P(rows_d), stream_handle())
    rows = rows_d[: ntl * 27].cpu().numpy().reshape(ntl, 27)
    valid = rows >= 0
    counts = valid.sum(axis=1)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    leaves = rows[valid].astype(np.int64)
    src_counts = np.where(valid, source_tree.leaf_counts[np.maximum(rows, 0)], 0).sum(axis=1)
    n_pairs = int((src_counts * target_tree.leaf_counts).sum())
    return NearFieldPlan(offsets, leaves, n_pairs)


_TABLES = {}


def _tables():
    key = torch.cuda.current_device()
    if key not in _TABLES:
        _TABLES[key] = (to_dev(class_transfer_table(), np.int32),
                        to_dev(transfer_offsets(), np.int8))
    return _TABLES[key]


def blas_level_plan(source_tree, target_tree, level: int):
    """Same plan as ``level_plan_from_buckets(bucket_level(...), ...)`` with
    the source table built on the device (kept there for the sweep)."""
    from .m2l_blas import TILE_TARGETS, BlasLevelPlan
    require_cuda()
    tcodes = target_tree.level_keys(level)
    n_t = tcodes.shape[0]
    cls = ((tcodes >> np.uint64(LEVEL_BITS)) & np.uint64(7)).astype(np.int64)
    order, tile_class = [], []
    for c in range(8):
        rows = np.flatnonzero(cls == c)
        nt = (rows.shape[0] + TILE_TARGETS - 1) // TILE_TARGETS
        pad = np.full(nt * TILE_TARGETS, -1, dtype=np.int64)
        pad[:rows.shape[0]] = rows
        order.append(pad)
        tile_class += [c] * nt
    slots = np.concatenate(order) if order else np.zeros(0, np.int64)
    n_slots = slots.shape[0]
    class_tv, offsets = _tables()
    src_d = torch.empty(max(n_slots, 1) * 189, dtype=torch.int32, device=_dev())
    slots_d = to_dev(slots, np.int32)
    nat.call("kifmm_blas_src_table", P(_dev_levels(target_tree)[level]), P(slots_d), n_slots,
             level, P(class_tv), P(offsets), P(_dev_levels(source_tree)[level]),
             source_tree.level_keys(level).shape[0], P(src_d), stream_handle())
    n_tiles = len(tile_class)
    src_t = src_d[: n_slots * 189].cpu().numpy().reshape(n_tiles, 189, TILE_TARGETS)
    src = np.ascontiguousarray(src_t.transpose(0, 2, 1)).reshape(n_slots, 189)
    plan = BlasLevelPlan(level, n_t, slots.astype(np.int32), np.asarray(tile_class, np.int32),
                         src, int((src >= 0).sum()))
    plan.src_dev = src_d[: max(n_slots, 1) * 189]
    return plan
