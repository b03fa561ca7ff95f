"""FFT-M2L: translations as circular convolutions on the 2p-per-side grid.

Host side (setup, reference semantics):
  * ``build_conv_grid`` - densities embed at lattice + p, potentials read at
    the lattice (reference ``m2l_fft.py:31-53``);
  * ``kernel_grid`` - kernel samples at ``-off - (j + 1 - p) h`` with the
    n-1 planes zeroed (``m2l_fft.py:56-80``);
  * ``precompute_fft_operators`` - ``khat[f, o, tau, sigma]``: spectrum of the
    flipped kernel grid for rel = 2 o + child[sigma] - child[tau], zero where
    the child pair is adjacent (``m2l_fft.py:133-161``).  Uses the same
    scipy.fft (pocketfft) calls so the spectra are bit-identical;
  * ``build_halo_plan`` - sibling-cluster slots and the 26-neighbour source
    cluster table (``m2l_fft.py:167-215``).

Device side: ``m2l_fft_level`` mirrors ``m2l_fft.py:218`` (host arrays in,
host array out) with forward transform, Hadamard and inverse transform on
the GPU (see :mod:`.device`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.fft

from .expansion import INNER_SCALE, INV_4PI, boundary_lattice, n_surface
from .octree import (Octree, child_index_codes, decode_codes, encode_anchors, halo_offsets,
                     parent_codes)


def _workers(workers):
    import os
    if workers is None:
        env = os.environ.get("KIFMM_THREADS", "").strip()
        try:
            n = int(env) if env else 0
        except ValueError:
            n = 0
        return n if n >= 1 else (os.cpu_count() or 1)
    return max(1, int(workers))


@dataclass
class ConvGrid:
    order: int
    n_grid: int
    n_freq: int
    embed_idx: np.ndarray
    read_idx: np.ndarray


def build_conv_grid(order: int) -> ConvGrid:
    n = 2 * order
    lat = boundary_lattice(order)

    def flat(a):
        return ((a[:, 0] * n + a[:, 1]) * n + a[:, 2]).astype(np.int64)

    return ConvGrid(order, n, n * n * (n // 2 + 1), flat(lat + order), flat(lat))


def kernel_grid(offset, order: int, dtype=np.float64, inner_scale=INNER_SCALE) -> np.ndarray:
    n = 2 * order
    h = inner_scale / (order - 1)
    off = np.asarray(offset, dtype=np.float64)
    j = np.arange(n, dtype=np.float64)
    cx, cy, cz = (-(off[a]) - (j + 1 - order) * h for a in range(3))
    r2 = (cx[:, None, None] ** 2 + cy[None, :, None] ** 2 + cz[None, None, :] ** 2)
    with np.errstate(divide="ignore"):
        vals = INV_4PI / np.sqrt(r2)
    vals[~np.isfinite(vals)] = 0.0
    vals[n - 1] = 0.0
    vals[:, n - 1] = 0.0
    vals[:, :, n - 1] = 0.0
    return vals.astype(dtype)


@dataclass
class M2lFftOperators:
    order: int
    grid: ConvGrid
    khat: np.ndarray          # (n_freq, 26, 8, 8) complex

    @property
    def n_freq(self) -> int:
        return self.grid.n_freq


_CHILD = np.array([[(i >> 2) & 1, (i >> 1) & 1, i & 1] for i in range(8)], dtype=np.int64)


def precompute_fft_operators(order: int, dtype=np.float64, inner_scale=INNER_SCALE,
                             workers=None) -> M2lFftOperators:
    grid = build_conv_grid(order)
    cdt = np.complex64 if np.dtype(dtype) == np.float32 else np.complex128
    halo = np.array(halo_offsets(), dtype=np.int64)
    rel = 2 * halo[:, None, None, :] + _CHILD[None, None, :, :] - _CHILD[None, :, None, :]
    admissible = np.abs(rel).max(axis=3) >= 2                # (26, tau, sigma)
    uniq, inv = np.unique(rel.reshape(-1, 3), axis=0, return_inverse=True)
    grids = np.stack([kernel_grid(u, order, dtype, inner_scale) for u in uniq])
    spec = scipy.fft.rfftn(np.flip(grids, axis=(1, 2, 3)), axes=(1, 2, 3),
                           workers=_workers(workers))
    spec = spec.reshape(uniq.shape[0], grid.n_freq).astype(cdt)
    inv = np.asarray(inv).reshape(26, 8, 8)
    khat = np.zeros((grid.n_freq, 26, 8, 8), dtype=cdt)
    o_i, t_i, s_i = np.nonzero(admissible)
    khat[:, o_i, t_i, s_i] = spec[inv[o_i, t_i, s_i]].T
    return M2lFftOperators(order, grid, np.ascontiguousarray(khat))


@dataclass
class HaloPlan:
    level: int
    n_src_clusters: int
    n_tgt_clusters: int
    src_slot: np.ndarray      # (n_src_boxes,) cluster*8 + child
    tgt_slot: np.ndarray      # (n_tgt_boxes,)
    halo: np.ndarray          # (n_tgt_clusters, 26) source cluster or -1
    src_color: np.ndarray = None   # (n_src_clusters,) coordinate parity class (x&1|y&1<<1|z&1<<2)
    tgt_color: np.ndarray = None   # (n_tgt_clusters,) same for the target clusters


def build_halo_plan(source_tree: Octree, target_tree: Octree, level: int) -> HaloPlan:
    sc, tc = source_tree.level_keys(level), target_tree.level_keys(level)
    sp, tp = parent_codes(sc), parent_codes(tc)
    spu, tpu = np.unique(sp), np.unique(tp)
    src_slot = np.searchsorted(spu, sp) * 8 + child_index_codes(sc)
    tgt_slot = np.searchsorted(tpu, tp) * 8 + child_index_codes(tc)
    anchors, _ = decode_codes(tpu)
    n = 1 << (level - 1)
    halo = np.full((tpu.shape[0], 26), -1, dtype=np.int64)
    for i, off in enumerate(halo_offsets()):
        cand = anchors + np.asarray(off)
        ok = np.all((cand >= 0) & (cand < n), axis=1)
        if not ok.any():
            continue
        rows = np.flatnonzero(ok)
        codes = encode_anchors(cand[rows], level - 1)
        pos = np.searchsorted(spu, codes)
        posc = np.minimum(pos, spu.shape[0] - 1)
        hit = spu[posc] == codes
        halo[rows[hit], i] = posc[hit]
    sa, _ = decode_codes(spu)
    return HaloPlan(level, int(spu.shape[0]), int(tpu.shape[0]), src_slot.astype(np.int64),
                    tgt_slot.astype(np.int64), halo, parity_class(sa), parity_class(anchors))


def parity_class(anchors: np.ndarray) -> np.ndarray:
    """Coordinate parity class x&1 | (y&1)<<1 | (z&1)<<2 of integer anchors."""
    a = np.asarray(anchors, dtype=np.int64).reshape(-1, 3)
    return (a[:, 0] & 1) | ((a[:, 1] & 1) << 1) | ((a[:, 2] & 1) << 2)


HAD_TILE = 256      # target clusters per tile (csrc/hadamard.cu TT)
HAD_UMAX = 600      # source slots per tile (UMAX); UMAX + class = absent (zero rows)
HAD_OFFSET_PARITY = parity_class(np.array(halo_offsets()))


@dataclass
class HadamardTiles:
    """Tile plan of a halo table for the tiled Hadamard kernel
    (csrc/hadamard.cu hadamard_tiled_kernel, which documents the layout).

    Per tile of consecutive target clusters: ``tcol`` places each target in
    a slot-table column of its parity class (column 32w + 4g + j <-> class
    g), ``src`` lists the distinct sources in shared-memory slots with
    slot % 8 = the source's parity class, and ``slots`` maps each (offset,
    column) to its source's slot.  At a fixed offset the 8 lane groups of a
    warp then read sources of 8 different classes -> 8 different banks."""
    begin: np.ndarray        # (n_tiles + 1,) target-cluster offsets
    src_off: np.ndarray      # (n_tiles + 1,) offsets into src
    src: np.ndarray          # per tile: source cluster of each slot (-1 = hole)
    slots: np.ndarray        # (n_tiles, 26, HAD_TILE) int16
    tcol: np.ndarray         # (n_tiles, HAD_TILE) int16 tile-local target, -1 = empty

    @property
    def n_tiles(self) -> int:
        return int(self.begin.shape[0] - 1)


def _slot_layout(u: np.ndarray, color: np.ndarray):
    """Slots for sorted distinct sources u: slot = 8 * (rank within its class) + class."""
    c = color[u]
    order = np.argsort(c, kind="stable")
    counts = np.bincount(c, minlength=8)
    rank = np.empty(u.shape[0], dtype=np.int64)
    rank[order] = np.arange(u.shape[0]) - np.repeat(np.cumsum(counts) - counts, counts)
    slot = 8 * rank + c
    n_slots = int(8 * counts.max()) if u.shape[0] else 0
    return slot, n_slots


def _columns(tc: np.ndarray, tile: int) -> np.ndarray:
    """Column of each tile-local target: the k-th target of class g goes to
    column 32 (k // 4) + 4 g + k % 4."""
    col = np.empty(tc.shape[0], dtype=np.int64)
    for g in range(8):
        idx = np.flatnonzero(tc == g)
        k = np.arange(idx.shape[0])
        col[idx] = 32 * (k // 4) + 4 * g + (k % 4)
    return col


def plan_hadamard_tiles(halo: np.ndarray, src_color: np.ndarray, tgt_color: np.ndarray,
                        tile: int = HAD_TILE, umax: int = HAD_UMAX) -> HadamardTiles:
    """Greedy tiling of the (Morton-ordered) target clusters: take up to
    ``tile`` consecutive clusters, halve while a parity class holds more than
    tile/8 of them or their sources need more than ``umax`` slots (a full
    256-cluster brick: 32 targets per class, 600 sources = 75 per class =
    exactly 600 slots)."""
    halo = np.asarray(halo, dtype=np.int64)
    src_color = np.asarray(src_color, dtype=np.int64)
    tgt_color = np.asarray(tgt_color, dtype=np.int64)
    n = halo.shape[0]
    per_class = tile // 8
    begin, src_off, srcs, slots, tcols = [0], [0], [], [], []
    b = 0
    while b < n:
        e = min(n, b + tile)
        while True:
            h = halo[b:e]
            tc = tgt_color[b:e]
            u = np.unique(h[h >= 0])
            slot, n_slots = _slot_layout(u, src_color)
            if (n_slots <= umax and np.bincount(tc, minlength=8).max() <= per_class) or e - b == 1:
                break
            e = b + (e - b) // 2
        table = np.full(n_slots, -1, dtype=np.int64)
        table[slot] = u
        loc = slot[np.searchsorted(u, h)] if u.shape[0] else np.zeros(h.shape, np.int64)
        absent = umax + (tc[:, None] ^ HAD_OFFSET_PARITY[None, :])
        loc = np.where(h < 0, absent, loc)
        col = _columns(tc, tile)
        sl = np.empty((26, tile), dtype=np.int16)
        col_class = (np.arange(tile) >> 2) & 7
        sl[:] = (umax + (col_class[None, :] ^ HAD_OFFSET_PARITY[:, None])).astype(np.int16)
        sl[:, col] = loc.T
        tcol = np.full(tile, -1, dtype=np.int16)
        tcol[col] = np.arange(e - b)
        srcs.append(table)
        slots.append(sl)
        tcols.append(tcol)
        begin.append(e)
        src_off.append(src_off[-1] + n_slots)
        b = e
    return HadamardTiles(np.asarray(begin, dtype=np.int64), np.asarray(src_off, dtype=np.int64),
                         np.concatenate(srcs).astype(np.int64) if srcs else np.zeros(0, np.int64),
                         np.stack(slots) if slots else np.zeros((0, 26, tile), np.int16),
                         np.stack(tcols) if tcols else np.zeros((0, tile), np.int16))


def m2l_fft_level(ops: M2lFftOperators, plan: HaloPlan, multipoles, level_scale: float = 1.0,
                  block_size: int = 32, threads=None) -> np.ndarray:
    """Drop-in for reference ``m2l_fft.m2l_fft_level`` (``m2l_fft.py:218-261``):
    host arrays in and out, forward FFT + Hadamard + inverse FFT on the GPU.
    ``block_size``/``threads`` are accepted for signature compatibility."""
    mult = np.asarray(multipoles)
    if mult.shape[2] != n_surface(ops.order):
        raise ValueError("the multipole width does not match the operator order")
    from . import device
    return device.m2l_fft_level_host(ops, plan, mult, level_scale)
