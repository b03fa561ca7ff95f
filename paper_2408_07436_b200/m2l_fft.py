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
    return HaloPlan(level, int(spu.shape[0]), int(tpu.shape[0]), src_slot.astype(np.int64),
                    tgt_slot.astype(np.int64), halo)


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
