"""Surface grids, kernel matrices and the regularised pseudo-inverses
(host-side setup numerics).

These build the unit-box operators that the device passes apply.  The
arithmetic is arranged so that every matrix is bit-identical to the one the
reference assembles on the same machine:

* surface lattices in lexicographic order, mapped as
  ``center + (lat/(p-1) - 0.5) * (scale*side)`` (reference ``expansion.py:34-52``);
* kernel entries ``K = fl(1/(4 pi)) / sqrt(r2)`` with ``r2`` summed x, y, z in
  the working dtype and ``K = 0`` on coincidence (``_hot.pyx:68-88``); IEEE
  division and square root give the same bits in numpy as in C;
* filtered-SVD pseudo-inverse ``V diag(s/(s^2+alpha)) U^T`` with a relative
  cutoff of 10 eps (``expansion.py:90-110``);
* inner scale 1.05, outer scale 2.95 (``expansion.py:27-28``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

INV_4PI = 0.079577471545947667884441881686257181
INNER_SCALE = 1.05
OUTER_SCALE = 2.95
CUTOFF_EPS_FACTOR = 10.0


def n_surface(order: int) -> int:
    return 6 * (order - 1) ** 2 + 2


def boundary_lattice(order: int) -> np.ndarray:
    """Integer points on the faces of [0, order-1]^3, lexicographic (i, j, k)."""
    if order < 2:
        raise ValueError("surface order must be at least 2")
    r = np.arange(order)
    g = np.array(np.meshgrid(r, r, r, indexing="ij")).reshape(3, -1).T
    face = ((g == 0) | (g == order - 1)).any(axis=1)
    return g[face]


def surface(order: int, center, side: float, scale: float, dtype=np.float64) -> np.ndarray:
    frac = boundary_lattice(order).astype(np.float64) / (order - 1) - 0.5
    pts = np.asarray(center, dtype=np.float64) + frac * (scale * side)
    return np.ascontiguousarray(pts, dtype=dtype)


def kernel_matrix(src, tgt, dtype=np.float64) -> np.ndarray:
    """Dense ``K[i, j] = K(tgt_i, src_j)`` in ``dtype`` (host, setup only)."""
    s = np.asarray(src, dtype=dtype).reshape(-1, 3)
    t = np.asarray(tgt, dtype=dtype).reshape(-1, 3)
    dx = t[:, 0:1] - s[None, :, 0]
    dy = t[:, 1:2] - s[None, :, 1]
    dz = t[:, 2:3] - s[None, :, 2]
    r2 = dx * dx + dy * dy
    r2 = r2 + dz * dz
    r = np.sqrt(r2)
    c = np.dtype(dtype).type(INV_4PI)
    with np.errstate(divide="ignore"):
        k = c / r
    k[r2 == 0] = 0
    return np.ascontiguousarray(k, dtype=dtype)


@dataclass
class RegularizedInverse:
    """``q = scale * V diag(inv_vals) U^T phi`` (filtered SVD pseudo-inverse)."""

    u: np.ndarray
    inv_vals: np.ndarray
    v: np.ndarray
    alpha: float
    cutoff: float

    @property
    def rank(self) -> int:
        return int(self.inv_vals.shape[0])

    def apply(self, phi, scale: float = 1.0):
        inner = self.u.T @ phi
        inner = (self.inv_vals[:, None] * inner) if inner.ndim == 2 else self.inv_vals * inner
        return (self.v @ inner) * scale


def tikhonov_pinv(k: np.ndarray, alpha: float = 0.0, cutoff: float | None = None) -> RegularizedInverse:
    if alpha < 0:
        raise ValueError("alpha must be nonnegative")
    if cutoff is None:
        cutoff = CUTOFF_EPS_FACTOR * float(np.finfo(k.dtype).eps)
    u, s, vt = np.linalg.svd(k, full_matrices=False)
    keep = (s >= cutoff * s[0]) if (s.shape[0] and s[0] > 0) else np.zeros(s.shape, bool)
    s = s[keep]
    inv = (s / (s * s + k.dtype.type(alpha))).astype(k.dtype)
    return RegularizedInverse(u=np.ascontiguousarray(u[:, keep]), inv_vals=inv,
                              v=np.ascontiguousarray(vt[keep].T), alpha=float(alpha),
                              cutoff=float(cutoff))


def child_offsets() -> np.ndarray:
    """Centres of the 8 children of a unit box at the origin (x bit highest)."""
    i = np.arange(8)
    bits = np.stack([(i >> 2) & 1, (i >> 1) & 1, i & 1], axis=1).astype(np.float64)
    return (bits - 0.5) / 2.0


class ExpansionOperators:
    """Unit-box upward/downward surfaces, pseudo-inverses and the child
    translation kernels (reference ``expansion.py:123-178``).

    ``m2m_kernels``: (n_check, 8*n_equiv) child equivalent -> parent check.
    ``l2l_kernels``: (8*n_check, n_equiv) parent equivalent -> child check.
    """

    def __init__(self, order_equiv: int, order_check: int | None = None, dtype=np.float64,
                 alpha: float = 0.0, cutoff: float | None = None,
                 inner_scale: float = INNER_SCALE, outer_scale: float = OUTER_SCALE):
        order_check = order_equiv if order_check is None else order_check
        if order_check < order_equiv:
            raise ValueError("check order must be at least the equivalent order")
        self.order_equiv, self.order_check = order_equiv, order_check
        self.dtype = np.dtype(dtype)
        self.alpha = alpha
        self.inner_scale, self.outer_scale = inner_scale, outer_scale
        self.n_equiv, self.n_check = n_surface(order_equiv), n_surface(order_check)
        o, dt = np.zeros(3), self.dtype
        self.up_equiv = surface(order_equiv, o, 1.0, inner_scale, dt)
        self.up_check = surface(order_check, o, 1.0, outer_scale, dt)
        self.down_equiv = surface(order_equiv, o, 1.0, outer_scale, dt)
        self.down_check = surface(order_check, o, 1.0, inner_scale, dt)
        self.up_inv = tikhonov_pinv(kernel_matrix(self.up_equiv, self.up_check, dt), alpha, cutoff)
        self.down_inv = tikhonov_pinv(kernel_matrix(self.down_equiv, self.down_check, dt), alpha, cutoff)
        cc = child_offsets()
        self.m2m_kernels = np.ascontiguousarray(np.hstack([
            kernel_matrix(surface(order_equiv, cc[i], 0.5, inner_scale, dt), self.up_check, dt)
            for i in range(8)]))
        self.l2l_kernels = np.ascontiguousarray(np.vstack([
            kernel_matrix(self.down_equiv, surface(order_check, cc[i], 0.5, inner_scale, dt), dt)
            for i in range(8)]))
