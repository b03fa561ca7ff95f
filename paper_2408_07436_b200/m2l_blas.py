"""BLAS-M2L: SVD-compressed field translation.

Host side (setup, reference semantics):
  * ``precompute`` builds the shared bases U (n_check x k), S (n_equiv x k)
    from one randomized SVD of the 316 unit-box translations side by side,
    the 316 cores C_t = U^T K_t S and their per-vector recompression
    C_t ~ ubar_t vbar_t^T with the singular values folded into vbar
    (reference ``m2l_blas.py:73-208``).  The seeded Gaussian sketch, the
    QR/SVD calls and the *absolute* finest-level cutoff
    ``sval * level_scale >= sigma_min`` are reproduced exactly so the
    operators are bit-identical on the same machine.
  * ``bucket_level`` groups the far-field pairs of a level by transfer
    vector (reference ``m2l_blas.py:232-258``).

Device side (the hot path): ``apply_level`` mirrors the reference
signature (``m2l_blas.py:270``) and runs the level on the GPU through the
C-ABI in :mod:`._native`; see :class:`BlasLevelPlan` for the
target-stationary layout the kernel consumes.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .expansion import INNER_SCALE, kernel_matrix, n_surface, surface
from .octree import (Octree, class_transfer_table, decode_codes, encode_anchors,
                     transfer_offsets, transfer_vector_index)

N_TRANSFER = 316


class CompressionError(RuntimeError):
    """No singular value survived the requested truncation."""


def assemble_translation(offset, order_equiv, order_check, dtype=np.float64,
                         inner_scale=INNER_SCALE) -> np.ndarray:
    """K_t: unit source box at anchor ``offset`` -> unit target box at 0."""
    src = surface(order_equiv, np.asarray(offset, dtype=np.float64), 1.0, inner_scale, dtype)
    tgt = surface(order_check, np.zeros(3), 1.0, inner_scale, dtype)
    return kernel_matrix(src, tgt, dtype)


def _fat_thin(order_equiv, order_check, dtype, inner_scale):
    blocks = [assemble_translation(o, order_equiv, order_check, dtype, inner_scale)
              for o in transfer_offsets()]
    fat = np.ascontiguousarray(np.hstack(blocks))
    if order_equiv == order_check:
        thin = np.ascontiguousarray(np.vstack([b.T for b in blocks]))
    else:
        thin = np.ascontiguousarray(np.vstack(
            [assemble_translation(o, order_check, order_equiv, dtype, inner_scale).T
             for o in transfer_offsets()]))
    return fat, thin


def rsvd(a: np.ndarray, rank: int, oversamples: int, rng):
    """Single-pass randomized SVD (Gaussian sketch -> QR -> small SVD)."""
    m, n = a.shape
    width = rank + oversamples
    if rank < 1:
        raise ValueError("rank must be positive")
    if width > min(m, n):
        raise ValueError(f"rank + oversamples = {width} exceeds min(shape) = {min(m, n)}")
    omega = rng.standard_normal((n, width)).astype(a.dtype, copy=False)
    basis, _ = np.linalg.qr(a @ omega)
    ub, sv, vt = np.linalg.svd(basis.T @ a, full_matrices=False)
    return (np.ascontiguousarray(basis @ ub[:, :rank]), sv[:rank].copy(),
            np.ascontiguousarray(vt[:rank].T))


@dataclass
class M2lBlasOperators:
    order_equiv: int
    order_check: int
    sigma_min: float
    level_scale: float
    u: np.ndarray
    s: np.ndarray
    svals_fat: np.ndarray
    svals_thin: np.ndarray
    ubar: list = field(default_factory=list)
    vbar: list = field(default_factory=list)
    cores: list | None = None

    @property
    def k(self) -> int:
        return int(self.u.shape[1])

    @property
    def ranks(self) -> np.ndarray:
        return np.array([u.shape[1] for u in self.ubar], dtype=np.int64)


def _keep_count(svals, sigma_min, level_scale):
    if svals.shape[0] == 0 or svals[0] <= 0:
        return 0
    if sigma_min <= 0:
        return int(svals.shape[0])
    return int(np.count_nonzero(svals * level_scale >= sigma_min))


def compress(order_equiv, order_check, sigma_min=1e-6, rank_estimate=None, oversamples=5,
             seed=0, dtype=np.float64, inner_scale=INNER_SCALE, level_scale=1.0,
             fat_thin=None) -> M2lBlasOperators:
    n_equiv = n_surface(order_equiv)
    rng = np.random.default_rng(seed)
    fat, thin = fat_thin if fat_thin is not None else _fat_thin(order_equiv, order_check,
                                                                dtype, inner_scale)
    full = min(min(fat.shape), min(thin.shape))
    if rank_estimate is None:
        rank_estimate = full - oversamples
    u_fat, s_fat, _ = rsvd(fat, max(1, min(rank_estimate, min(fat.shape) - oversamples)),
                           oversamples, rng)
    if order_equiv == order_check:
        s_basis, s_thin = u_fat, s_fat
    else:
        _, s_thin, s_basis = rsvd(thin, max(1, min(rank_estimate, min(thin.shape) - oversamples)),
                                  oversamples, rng)
    k = min(_keep_count(s_fat, sigma_min, level_scale), _keep_count(s_thin, sigma_min, level_scale))
    if k == 0:
        raise CompressionError("sigma_min truncated every singular value")
    u = np.ascontiguousarray(u_fat[:, :k])
    s = np.ascontiguousarray(s_basis[:, :k])
    proj = u.T @ fat
    cores = [np.ascontiguousarray(proj[:, i * n_equiv:(i + 1) * n_equiv] @ s)
             for i in range(N_TRANSFER)]
    return M2lBlasOperators(order_equiv, order_check, sigma_min, level_scale, u, s,
                            s_fat.copy(), s_thin.copy(), cores=cores)


def recompress(ops: M2lBlasOperators, sigma_min=None) -> M2lBlasOperators:
    if ops.cores is None:
        raise ValueError("operators carry no cores to recompress")
    cut = ops.sigma_min if sigma_min is None else sigma_min
    ops.ubar, ops.vbar = [], []
    for c in ops.cores:
        ub, sv, vt = np.linalg.svd(c, full_matrices=False)
        positive = sv.shape[0] > 0 and sv[0] > 0
        if positive and cut > 0:
            kt = int(np.count_nonzero(sv * ops.level_scale >= cut))
        else:
            kt = sv.shape[0] if positive else 0
        ops.ubar.append(np.ascontiguousarray(ub[:, :kt]))
        ops.vbar.append(np.ascontiguousarray(vt[:kt].T * sv[:kt]))
    return ops


def precompute(order_equiv, order_check, sigma_min=1e-6, rank_estimate=None, oversamples=5,
               seed=0, dtype=np.float64, inner_scale=INNER_SCALE,
               level_scale=1.0) -> M2lBlasOperators:
    return recompress(compress(order_equiv, order_check, sigma_min, rank_estimate, oversamples,
                               seed, dtype, inner_scale, level_scale))


# ------------------------------------------------------------- pair buckets
@dataclass
class TransferBuckets:
    """Far-field pairs of a level grouped by transfer vector; ``pairs[i]`` is
    ``(source_rows, target_rows)`` or None.  Targets are distinct in a bucket."""

    level: int
    pairs: list

    @property
    def n_nonempty(self) -> int:
        return sum(p is not None for p in self.pairs)


def bucket_level(source_tree: Octree, target_tree: Octree, level: int) -> TransferBuckets:
    tcodes = target_tree.level_keys(level)
    pairs: list = [None] * N_TRANSFER
    if tcodes.shape[0] == 0 or source_tree.level_keys(level).shape[0] == 0:
        return TransferBuckets(level, pairs)
    anchors, _ = decode_codes(tcodes)
    n = 1 << level
    half = anchors >> 1
    for i, off in enumerate(transfer_offsets()):
        cand = anchors + off
        ok = np.all((cand >= 0) & (cand < n) & (np.abs((cand >> 1) - half) <= 1), axis=1)
        if not ok.any():
            continue
        rows_t = np.flatnonzero(ok)
        rows_s = source_tree.lookup(encode_anchors(cand[rows_t], level), level)
        hit = rows_s >= 0
        if hit.any():
            pairs[i] = (rows_s[hit].astype(np.int64), rows_t[hit].astype(np.int64))
    return TransferBuckets(level, pairs)


def _expand_rows(rows: np.ndarray, n_rhs: int) -> np.ndarray:
    if n_rhs == 1:
        return rows
    return (rows[:, None] * n_rhs + np.arange(n_rhs)[None, :]).ravel()


# ------------------------------------------------- device level plan (ours)
TILE_TARGETS = 128


@dataclass
class BlasLevelPlan:
    """Target-stationary layout of one level's far field for the device.

    Targets are grouped by parity class (anchor bits), because every target
    of a class meets the same 189 transfer vectors (``class_transfer_table``).
    ``tile_targets[i]`` is the target row (or -1 padding) of slot ``i``;
    ``tile_class[t]`` the class of tile ``t``; ``src[i, j]`` the source row
    met by slot ``i`` through the class's j-th vector (or -1).  The kernel
    walks j in ascending canonical order, which fixes the accumulation
    order: results are deterministic run to run.
    """

    level: int
    n_targets: int
    tile_targets: np.ndarray   # (n_tiles*TILE,) int32
    tile_class: np.ndarray     # (n_tiles,) int32
    src: np.ndarray            # (n_tiles*TILE, 189) int32
    n_pairs: int


def infer_target_classes(buckets: TransferBuckets, n_targets: int) -> np.ndarray:
    """Parity class of each target row from the offsets it meets: an offset
    component +3 forces an even anchor, -3 an odd one; unconstrained axes
    default to even (both classes then list every offset the target meets)."""
    offs = transfer_offsets()
    odd = np.zeros((n_targets, 3), dtype=bool)
    even = np.zeros((n_targets, 3), dtype=bool)
    for i, pr in enumerate(buckets.pairs):
        if pr is None:
            continue
        rt = pr[1]
        even[rt] |= offs[i] == 3
        odd[rt] |= offs[i] == -3
    if np.any(odd & even):
        raise ValueError("bucket pairs are inconsistent with any parity class")
    bits = odd.astype(np.int64)
    return (bits[:, 0] << 2) | (bits[:, 1] << 1) | bits[:, 2]


def level_plan_from_buckets(buckets: TransferBuckets, n_targets: int,
                            target_classes=None, owned=None) -> BlasLevelPlan:
    """``owned`` (optional (lo, hi) target-row range): tile only those
    targets (a rank of the partitioned evaluate sweeps its own tiles)."""
    if target_classes is None:
        target_classes = infer_target_classes(buckets, n_targets)
    table = class_transfer_table()                      # (8, 189)
    pos_in_class = np.full((8, N_TRANSFER), -1, dtype=np.int64)
    for c in range(8):
        pos_in_class[c, table[c]] = np.arange(189)
    cls = np.asarray(target_classes, dtype=np.int64)
    order = []
    tile_class = []
    keep = np.ones(cls.shape[0], dtype=bool)
    if owned is not None:
        keep[:] = False
        keep[owned[0]:owned[1]] = True
    for c in range(8):
        rows = np.flatnonzero((cls == c) & keep)
        n_t = (rows.shape[0] + TILE_TARGETS - 1) // TILE_TARGETS
        pad = np.full(n_t * TILE_TARGETS, -1, dtype=np.int64)
        pad[:rows.shape[0]] = rows
        order.append(pad)
        tile_class += [c] * n_t
    slots = np.concatenate(order) if order else np.zeros(0, np.int64)
    slot_of_target = np.full(n_targets, -1, dtype=np.int64)
    valid = slots >= 0
    slot_of_target[slots[valid]] = np.flatnonzero(valid)
    src = np.full((slots.shape[0], 189), -1, dtype=np.int32)
    n_pairs = 0
    for i, pr in enumerate(buckets.pairs):
        if pr is None:
            continue
        rs, rt = pr
        j = pos_in_class[cls[rt], i]
        if np.any(j < 0):
            raise ValueError("bucket pair inadmissible for its target parity class")
        sl = slot_of_target[rt]
        if np.any(sl < 0):
            raise ValueError("bucket pair targets a row outside the planned targets")
        src[sl, j] = rs
        n_pairs += rs.shape[0]
    return BlasLevelPlan(buckets.level, n_targets, slots.astype(np.int32),
                         np.asarray(tile_class, dtype=np.int32), src, n_pairs)


def dense_cores(ops: M2lBlasOperators, dtype) -> np.ndarray:
    """(316, k, k) contracted recompressed cores D_t = ubar_t vbar_t^T, formed
    in float64 and rounded once to ``dtype``; row = output (check-basis)
    index, column = input (source-basis) index."""
    k = ops.k
    out = np.zeros((N_TRANSFER, k, k), dtype=np.float64)
    for i in range(N_TRANSFER):
        if ops.ubar[i].shape[1]:
            out[i] = ops.ubar[i].astype(np.float64) @ ops.vbar[i].astype(np.float64).T
    return out.astype(dtype)


def apply_level(ops: M2lBlasOperators, buckets: TransferBuckets, multipoles, n_targets: int,
                level_scale: float = 1.0, counter: list | None = None,
                strategy: str = "serial", threads: int = 1) -> np.ndarray:
    """Drop-in for reference ``m2l_blas.apply_level`` (``m2l_blas.py:270-326``):
    host arrays in, host array out, all arithmetic on the GPU.

    ``strategy``/``threads`` are accepted for signature compatibility; the
    device kernel is one deterministic target-stationary sweep.  ``counter``
    receives the number of device launches of the level (projection, fused
    bucket sweep, expansion).
    """
    from . import device
    return device.apply_level_host(ops, buckets, multipoles, n_targets, level_scale, counter)
