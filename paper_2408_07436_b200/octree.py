"""Morton-coded uniform octree (host-side setup geometry).

Semantics follow the reference tree so that every plan the device consumes
(level key arrays, leaf ranges, point permutation) is identical:

* key layout: interleaved anchor bits, x most significant, sitting above a
  5-bit level field (``octree.py:1-9``, ``octree.py:67-71`` of the reference);
* domain: tight bounding cube of both clouds widened by a relative 1e-5
  margin (``octree.py:255-264``);
* leaf encoding clamps points on the upper faces into the last box row
  (``octree.py:274-288``);
* points are stably sorted by leaf code and empty branches are pruned
  (``octree.py:303-329``).

The implementation here is our own (byte-table interleave, vectorised
neighbour and interaction-list generation); it is setup-time host work and
never on the evaluate path.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

MAX_DEPTH = 16
LEVEL_BITS = 5
DOMAIN_MARGIN = 1e-5


class DomainError(ValueError):
    """A point lies outside the tree domain."""


class LevelError(ValueError):
    """A key operation was asked for at an invalid level."""


# ---------------------------------------------------------------- interleave
def _make_spread_table() -> np.ndarray:
    # spread 8 input bits three apart: bit b -> bit 3b
    tab = np.zeros(256, dtype=np.uint64)
    for v in range(256):
        out = 0
        for b in range(8):
            if v >> b & 1:
                out |= 1 << (3 * b)
        tab[v] = out
    return tab


_SPREAD8 = _make_spread_table()


def _spread16(v: np.ndarray) -> np.ndarray:
    v = np.asarray(v, dtype=np.uint64)
    lo = _SPREAD8[(v & np.uint64(0xFF)).astype(np.intp)]
    hi = _SPREAD8[((v >> np.uint64(8)) & np.uint64(0xFF)).astype(np.intp)]
    return lo | (hi << np.uint64(24))


def _gather16(v: np.ndarray) -> np.ndarray:
    v = np.asarray(v, dtype=np.uint64)
    out = np.zeros(v.shape, dtype=np.uint64)
    for b in range(16):
        out |= ((v >> np.uint64(3 * b)) & np.uint64(1)) << np.uint64(b)
    return out


def encode_anchors(anchors, level) -> np.ndarray:
    """Codes of integer anchors ``(n, 3)`` at ``level`` (uint64)."""
    a = np.asarray(anchors, dtype=np.int64).reshape(-1, 3).astype(np.uint64)
    il = (_spread16(a[:, 0]) << np.uint64(2)) | (_spread16(a[:, 1]) << np.uint64(1)) \
        | _spread16(a[:, 2])
    return (il << np.uint64(LEVEL_BITS)) | np.uint64(level)


def decode_codes(codes):
    """``(anchors (n,3) int64, levels (n,) int64)`` of uint64 codes."""
    c = np.asarray(codes, dtype=np.uint64)
    levels = (c & np.uint64((1 << LEVEL_BITS) - 1)).astype(np.int64)
    il = c >> np.uint64(LEVEL_BITS)
    xyz = [_gather16(il >> np.uint64(s)).astype(np.int64) for s in (2, 1, 0)]
    return np.stack(xyz, axis=1), levels


def parent_codes(codes) -> np.ndarray:
    c = np.asarray(codes, dtype=np.uint64)
    lvl = c & np.uint64((1 << LEVEL_BITS) - 1)
    return ((c >> np.uint64(LEVEL_BITS + 3)) << np.uint64(LEVEL_BITS)) | (lvl - np.uint64(1))


def child_index_codes(codes) -> np.ndarray:
    """Position among siblings (x bit 4, y bit 2, z bit 1)."""
    c = np.asarray(codes, dtype=np.uint64)
    return ((c >> np.uint64(LEVEL_BITS)) & np.uint64(7)).astype(np.int64)


# --------------------------------------------------------------------- keys
@dataclass(frozen=True)
class MortonKey:
    anchor: tuple
    level: int

    def __post_init__(self):
        if not 0 <= self.level <= MAX_DEPTH:
            raise LevelError(f"level {self.level} outside [0, {MAX_DEPTH}]")
        n = 1 << self.level
        if any(not 0 <= int(a) < n for a in self.anchor):
            raise DomainError(f"anchor {self.anchor} outside the level-{self.level} grid")
        object.__setattr__(self, "anchor", tuple(int(a) for a in self.anchor))

    @property
    def code(self) -> int:
        return int(encode_anchors(np.array([self.anchor]), self.level)[0])

    @classmethod
    def from_code(cls, code) -> "MortonKey":
        a, l = decode_codes(np.array([code], dtype=np.uint64))
        return cls(tuple(int(v) for v in a[0]), int(l[0]))

    def parent(self) -> "MortonKey":
        if self.level == 0:
            raise LevelError("the root has no parent")
        return MortonKey(tuple(a >> 1 for a in self.anchor), self.level - 1)

    def child_index(self) -> int:
        x, y, z = self.anchor
        return (x & 1) << 2 | (y & 1) << 1 | (z & 1)

    def __lt__(self, other: "MortonKey") -> bool:
        return self.code < other.code


@lru_cache(maxsize=1)
def transfer_offsets() -> np.ndarray:
    """The 316 far-field anchor offsets (source - target), lexicographic
    over [-3, 3]^3 with Chebyshev norm >= 2 (reference ``octree.py:210-216``)."""
    offs = [o for o in itertools.product(range(-3, 4), repeat=3) if max(map(abs, o)) >= 2]
    out = np.array(offs, dtype=np.int64)
    out.setflags(write=False)
    return out


@lru_cache(maxsize=1)
def transfer_vector_index() -> dict:
    return {tuple(int(v) for v in o): i for i, o in enumerate(transfer_offsets())}


@lru_cache(maxsize=1)
def halo_offsets() -> tuple:
    """The 26 parent-neighbour offsets, lexicographic (``octree.py:224-228``)."""
    return tuple(o for o in itertools.product((-1, 0, 1), repeat=3) if o != (0, 0, 0))


def neighbors(key: MortonKey) -> list:
    """Adjacent same-level boxes inside the domain, sorted by code."""
    n = 1 << key.level
    out = []
    for off in halo_offsets():
        c = tuple(a + o for a, o in zip(key.anchor, off))
        if all(0 <= v < n for v in c):
            out.append(MortonKey(c, key.level))
    return sorted(out)


def interaction_list(key: MortonKey) -> list:
    """Children of the parent's neighbours that are not adjacent to ``key``."""
    if key.level < 2:
        return []
    out = []
    for pn in neighbors(key.parent()):
        px, py, pz = (2 * a for a in pn.anchor)
        for i in range(8):
            ch = (px + (i >> 2), py + ((i >> 1) & 1), pz + (i & 1))
            if max(abs(c - a) for c, a in zip(ch, key.anchor)) >= 2:
                out.append(MortonKey(ch, key.level))
    return sorted(out)


@lru_cache(maxsize=8)
def class_transfer_table() -> np.ndarray:
    """(8, 189) transfer-vector indices valid for each parity class.

    A target at anchor ``a`` meets offset ``o`` (per axis) iff the source's
    parent is adjacent to its own: o in [-2, 3] for even a, [-3, 2] for odd
    a.  Each class therefore has exactly 6^3 - 27 = 189 admissible vectors,
    listed in ascending canonical (lexicographic) order.
    """
    offs = transfer_offsets()
    rows = []
    for cls in range(8):
        par = np.array([(cls >> 2) & 1, (cls >> 1) & 1, cls & 1])
        lo = np.where(par == 0, -2, -3)
        hi = np.where(par == 0, 3, 2)
        ok = np.all((offs >= lo) & (offs <= hi), axis=1)
        idx = np.flatnonzero(ok)
        assert idx.shape[0] == 189
        rows.append(idx)
    return np.stack(rows).astype(np.int64)


# ------------------------------------------------------------ domain + tree
@dataclass(frozen=True)
class Domain:
    origin: tuple
    side: float

    @classmethod
    def from_points(cls, points, margin: float = DOMAIN_MARGIN) -> "Domain":
        p = np.asarray(points, dtype=np.float64).reshape(-1, 3)
        lo, hi = p.min(axis=0), p.max(axis=0)
        extent = float((hi - lo).max())
        side = extent * (1.0 + margin) if extent > 0 else 1.0
        origin = (lo + hi) / 2.0 - side / 2.0
        return cls(tuple(float(v) for v in origin), side)

    def box_side(self, level: int) -> float:
        return self.side / (1 << level)

    def box_center(self, key: MortonKey) -> np.ndarray:
        h = self.box_side(key.level)
        return np.asarray(self.origin, dtype=np.float64) + (np.asarray(key.anchor) + 0.5) * h


def encode_points(points, depth: int, domain: Domain) -> np.ndarray:
    p = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    frac = (p - np.asarray(domain.origin, dtype=np.float64)) / domain.side
    bad = np.any((frac < 0) | (frac > 1), axis=1)
    if bad.any():
        raise DomainError(f"point {p[int(np.argmax(bad))]} lies outside the domain")
    n = 1 << depth
    anchors = np.minimum((frac * n).astype(np.int64), n - 1)
    return encode_anchors(anchors, depth)


class Octree:
    """Pruned uniform octree of one point cloud, points in leaf-Morton order."""

    def __init__(self, points, depth: int, domain: Domain | None = None):
        p = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        if p.shape[0] < 1:
            raise ValueError("a tree needs at least one point")
        if not 1 <= depth <= MAX_DEPTH:
            raise LevelError(f"depth {depth} outside [1, {MAX_DEPTH}]")
        self.depth = depth
        self.domain = domain if domain is not None else Domain.from_points(p)
        codes = encode_points(p, depth, self.domain)
        self.perm = np.argsort(codes, kind="stable")
        sc = codes[self.perm]
        self.x = np.ascontiguousarray(p[self.perm, 0])
        self.y = np.ascontiguousarray(p[self.perm, 1])
        self.z = np.ascontiguousarray(p[self.perm, 2])
        self.n_points = p.shape[0]
        # run-length encode the sorted leaf codes
        brk = np.flatnonzero(np.r_[True, sc[1:] != sc[:-1]])
        leaves = sc[brk]
        self.leaf_starts = brk.astype(np.int64)
        self.leaf_counts = np.diff(np.r_[brk, sc.shape[0]]).astype(np.int64)
        self.levels = [None] * (depth + 1)
        self.levels[depth] = leaves
        for lvl in range(depth - 1, -1, -1):
            self.levels[lvl] = np.unique(parent_codes(self.levels[lvl + 1]))

    @classmethod
    def from_arrays(cls, depth, domain, perm, sorted_points, leaf_starts, leaf_counts, levels):
        """A tree from already-built arrays (device_setup.octree): points in
        leaf-Morton order, the permutation, leaf runs and per-level codes."""
        t = cls.__new__(cls)
        t.depth = depth
        t.domain = domain
        t.perm = np.asarray(perm, dtype=np.int64)
        sp = np.asarray(sorted_points, dtype=np.float64).reshape(-1, 3)
        t.x = np.ascontiguousarray(sp[:, 0])
        t.y = np.ascontiguousarray(sp[:, 1])
        t.z = np.ascontiguousarray(sp[:, 2])
        t.n_points = sp.shape[0]
        t.leaf_starts = np.asarray(leaf_starts, dtype=np.int64)
        t.leaf_counts = np.asarray(leaf_counts, dtype=np.int64)
        t.levels = [np.asarray(l, dtype=np.uint64) for l in levels]
        return t

    @property
    def leaves(self) -> np.ndarray:
        return self.levels[self.depth]

    def level_keys(self, level: int) -> np.ndarray:
        if not 0 <= level <= self.depth:
            raise LevelError(f"level {level} outside [0, {self.depth}]")
        return self.levels[level]

    def key_position(self, code, level: int) -> int:
        arr = self.levels[level]
        i = int(np.searchsorted(arr, np.uint64(code)))
        return i if i < arr.shape[0] and arr[i] == np.uint64(code) else -1

    def lookup(self, codes, level: int) -> np.ndarray:
        """Row of each code in the level array, -1 where pruned (vectorised)."""
        arr = self.levels[level]
        codes = np.asarray(codes, dtype=np.uint64)
        pos = np.searchsorted(arr, codes)
        posc = np.minimum(pos, arr.shape[0] - 1)
        hit = arr[posc] == codes
        return np.where(hit, posc, -1).astype(np.int64)

    def leaf_slice(self, code) -> slice:
        i = self.key_position(code, self.depth)
        if i < 0:
            raise KeyError(code)
        s = int(self.leaf_starts[i])
        return slice(s, s + int(self.leaf_counts[i]))

    def points_in_leaf(self, code) -> np.ndarray:
        sl = self.leaf_slice(code)
        return np.stack([self.x[sl], self.y[sl], self.z[sl]], axis=1)
