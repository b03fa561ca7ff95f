"""Host-side plans of the near-field (P2P) passes.

* :func:`mutual_slots` - the partial-sum slot layout of the mutual near field
  (``csrc/p2p_mutual.cu``): when the source and target clouds are one point
  set, every unordered pair of adjacent leaves is evaluated once, by the
  lower leaf, and the column sums it produces for the upper leaf land in a
  slot of that leaf reserved for it.  The reference evaluates each ordered
  pair (``engine.py:224-256`` plan, ``_hot.pyx:91-138`` loop).
* :func:`f32_cross_leaf_coincident` - whether rounding to float32 makes a
  target coincide with a source of ANOTHER leaf; the unguarded inner loops
  assume it does not (the reference guards every pair, ``_hot.pyx:44-50``),
  so the device path switches to the guarded variants when it does.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class MutualSlots:
    """Slot layout of the mutual near field, per leaf b (n_b points,
    nlow_b adjacent leaves below b): slot 0 holds b's own row sums, slot s
    (1 <= s <= nlow_b) the column sums of b's near-list entry s (a lower
    neighbour), at ``base[b] + s * n_b + t``."""

    base: np.ndarray         # (n_leaves,) int32
    nlow: np.ndarray         # (n_leaves,) int32
    near_dst: np.ndarray     # (len(near.leaves),) int32: base[B] + slot * n_B for upper entries, else -1
    total: int               # floats per right-hand side

    def pack(self, near_offsets, near_leaves, leaf_starts, leaf_counts) -> np.ndarray:
        """(len(near.leaves), 4) int32 device table of csrc/p2p_mutual.cu:
        (start, count, dst, leaf) per near entry; the own entry (first of
        each list) carries the leaf's slot base as dst."""
        lv = np.asarray(near_leaves, dtype=np.int64)
        off = np.asarray(near_offsets, dtype=np.int64)
        dst = self.near_dst.astype(np.int64).copy()
        nonempty = np.diff(off) > 0
        dst[off[:-1][nonempty]] = self.base[np.flatnonzero(nonempty)]
        out = np.stack([np.asarray(leaf_starts, np.int64)[lv], np.asarray(leaf_counts, np.int64)[lv],
                        dst, lv], axis=1)
        return np.ascontiguousarray(out.astype(np.int32))


def mutual_order(near_offsets, near_leaves, leaf_counts) -> np.ndarray:
    """Leaves by descending mutual-pass work (targets x (own + upper
    columns)): the launch order of csrc/p2p_mutual.cu (longest first)."""
    off = np.asarray(near_offsets, dtype=np.int64)
    lv = np.asarray(near_leaves, dtype=np.int64)
    n = np.asarray(leaf_counts, dtype=np.int64)
    owner = np.repeat(np.arange(n.shape[0]), np.diff(off))
    up = lv > owner
    cols = np.bincount(owner[up], weights=n[lv[up]], minlength=n.shape[0])
    work = n * (cols + n)
    return np.argsort(-work, kind="stable").astype(np.int32)


def mutual_slots(near_offsets, near_leaves, leaf_counts) -> MutualSlots:
    off = np.asarray(near_offsets, dtype=np.int64)
    lv = np.asarray(near_leaves, dtype=np.int64)
    n = np.asarray(leaf_counts, dtype=np.int64)
    nl = n.shape[0]
    owner = np.repeat(np.arange(nl, dtype=np.int64), np.diff(off))
    pos = np.arange(lv.shape[0], dtype=np.int64) - off[owner]
    if lv.size and not np.all(lv[off[:-1][np.diff(off) > 0]] == np.flatnonzero(np.diff(off) > 0)):
        raise ValueError("near lists must start with the leaf itself")
    lower = lv < owner
    upper = lv > owner
    nlow = np.bincount(owner[lower], minlength=nl).astype(np.int64)
    # the lower entries of a near list are its entries 1..nlow (ascending order)
    if np.any(pos[lower] > nlow[owner[lower]]):
        raise ValueError("near lists must list neighbours in ascending leaf order")
    sizes = n * (1 + nlow)
    base = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    total = int(base[-1])
    if total >= 2 ** 31:
        raise ValueError("mutual near-field slots exceed int32 indexing")
    # slot of A in B's list, for every upper entry (A, B) of A's list
    key_low = owner[lower] * nl + lv[lower]            # (B, A) from B's side
    order = np.argsort(key_low, kind="stable")
    key_up = lv[upper] * nl + owner[upper]             # (B, A) from A's side
    hit = np.searchsorted(key_low[order], key_up)
    if key_up.size and (np.any(hit >= key_low.size) or
                        np.any(key_low[order][np.minimum(hit, key_low.size - 1)] != key_up)):
        raise ValueError("near lists are not symmetric (sources and targets differ)")
    slot = pos[lower][order][hit]
    dst = np.full(lv.shape[0], -1, dtype=np.int64)
    dst[upper] = base[lv[upper]] + slot * n[lv[upper]]
    return MutualSlots(base=base[:-1].astype(np.int32), nlow=nlow.astype(np.int32),
                       near_dst=dst.astype(np.int32), total=total)


def _f32_bits(tree):
    return (np.ascontiguousarray(tree.x, dtype=np.float32).view(np.uint32),
            np.ascontiguousarray(tree.y, dtype=np.float32).view(np.uint32),
            np.ascontiguousarray(tree.z, dtype=np.float32).view(np.uint32))


def f32_cross_leaf_coincident(target_tree, source_tree) -> bool:
    """True when some target and some source lie in different leaves (leaf
    Morton codes) yet have identical float32 coordinates."""
    tx, ty, tz = _f32_bits(target_tree)
    sx, sy, sz = _f32_bits(source_tree)
    tcode = np.repeat(np.asarray(target_tree.leaves, dtype=np.uint64), target_tree.leaf_counts)
    scode = np.repeat(np.asarray(source_tree.leaves, dtype=np.uint64), source_tree.leaf_counts)
    same = source_tree is target_tree or (
        tx.shape == sx.shape and np.array_equal(tx, sx) and np.array_equal(ty, sy)
        and np.array_equal(tz, sz) and np.array_equal(tcode, scode))
    if same:
        x, y, z, code = tx, ty, tz, tcode
    else:
        x, y, z = (np.concatenate(p) for p in ((tx, sx), (ty, sy), (tz, sz)))
        code = np.concatenate([tcode, scode])
    xy = (x.astype(np.uint64) << np.uint64(32)) | y.astype(np.uint64)
    order = np.argsort(xy, kind="stable")
    s = xy[order]
    dup = np.flatnonzero(s[1:] == s[:-1])
    if dup.size == 0:
        return False
    cand = np.unique(np.concatenate([order[dup], order[dup + 1]]))
    key = np.stack([x[cand], y[cand], z[cand]], axis=1)
    o = np.lexsort((key[:, 2], key[:, 1], key[:, 0]))
    k, c = key[o], code[cand][o]
    eq = np.all(k[1:] == k[:-1], axis=1)
    # runs of equal coordinates spanning two leaves
    return bool(np.any(eq & (c[1:] != c[:-1])))
