"""FMM engine: configuration, host-side setup and the device-resident evaluate.

Public surface mirrors the reference ``kifmm3d.engine`` (``engine.py:32-459``):
``FmmConfig`` (same fields, defaults and validation), ``setup(sources,
targets, config) -> FmmInstance``, ``FmmInstance.evaluate(charges)``,
``attach_charges``, ``relative_error`` and ``operator_timings``.

``setup`` runs on the host (trees, operators, per-level plans - setup-time
work the reference also does on the host) but builds the near-field plan as
a vectorised source-leaf CSR instead of the reference's per-leaf Python
loop (``engine.py:224-256``), so a 1M-point setup takes seconds, not minutes.
``evaluate`` runs every pass on the GPU (:mod:`.device`): there is no host
compute path.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

from . import m2l_blas, m2l_fft
from .expansion import ExpansionOperators, surface
from .octree import (MAX_DEPTH, Domain, MortonKey, Octree, child_index_codes, decode_codes,
                     encode_anchors, halo_offsets, parent_codes)

OPERATOR_NAMES = ("p2m", "m2m", "m2l", "l2l", "l2p", "p2p")


class ConfigError(ValueError):
    """An FmmConfig field is out of range or inconsistent."""


def _resolve_threads(threads=None) -> int:
    import os
    if threads is not None:
        return max(1, int(threads))
    env = os.environ.get("KIFMM_THREADS", "").strip()
    try:
        n = int(env) if env else 0
    except ValueError:
        n = 0
    return n if n >= 1 else (os.cpu_count() or 1)


@dataclass
class FmmConfig:
    """Engine parameters; same fields and defaults as reference ``engine.py:32-55``."""

    depth: int = 3
    order_equiv: int = 6
    order_check: int | None = None
    backend: str = "blas"
    precision: str = "f64"
    sigma_min: float = 1e-6
    oversamples: int = 5
    rank_estimate: int | None = None
    alpha: float = 0.0
    svd_cutoff: float | None = None
    block_size: int = 32
    n_rhs: int = 1
    seed: int = 0
    threads: int | None = None
    m2l_strategy: str | None = None
    p2m_block: int = 4
    m2m_block: int = 2
    inner_scale: float = 1.05
    outer_scale: float = 2.95

    def __post_init__(self):
        self.validate()

    def validate(self):
        checks = [
            (2 <= self.depth <= MAX_DEPTH, f"depth must lie in [2, {MAX_DEPTH}]"),
            (self.order_equiv >= 2, "the equivalent surface order must be at least 2"),
            (self.resolved_order_check() >= self.order_equiv,
             "the check order must be at least the equivalent order"),
            (self.backend in ("blas", "fft"), f"unknown backend {self.backend!r}"),
            (self.backend != "fft" or self.resolved_order_check() == self.order_equiv,
             "the FFT back end needs equal surface orders"),
            (self.precision in ("f32", "f64"), f"unknown precision {self.precision!r}"),
            (self.sigma_min >= 0, "sigma_min must be nonnegative"),
            (self.alpha >= 0, "alpha must be nonnegative"),
            (self.oversamples >= 1, "oversamples must be at least 1"),
            (self.block_size >= 1, "block_size must be at least 1"),
            (self.n_rhs >= 1, "n_rhs must be at least 1"),
            (self.p2m_block >= 1 and self.m2m_block >= 1, "sibling block sizes must be at least 1"),
            (self.m2l_strategy in (None, "serial", "bucket-threads"),
             f"unknown m2l strategy {self.m2l_strategy!r}"),
            (0 < self.inner_scale < self.outer_scale, "surface scales must satisfy 0 < inner < outer"),
        ]
        for ok, msg in checks:
            if not ok:
                raise ConfigError(msg)

    @property
    def dtype(self):
        return np.float32 if self.precision == "f32" else np.float64

    def resolved_order_check(self) -> int:
        return self.order_equiv if self.order_check is None else self.order_check

    def resolved_threads(self) -> int:
        return _resolve_threads(self.threads)

    def resolved_m2l_strategy(self) -> str:
        if self.m2l_strategy is not None:
            return self.m2l_strategy
        return "serial" if self.resolved_threads() <= 16 else "bucket-threads"


class ErrorStats(NamedTuple):
    error: float
    n_excluded: int


@dataclass
class NearFieldPlan:
    """Per target leaf, the source leaves of its near field: own leaf first,
    then adjacent leaves by Morton code (reference order, engine.py:231-240)."""

    offsets: np.ndarray      # (n_tleaves + 1,) int64
    leaves: np.ndarray       # (sum,) int64 source-leaf rows
    n_pairs: int             # sum over target leaves of n_targets * n_near_sources

    def source_rows(self, source_tree: Octree):
        """Expand to the reference's gathered-row CSR (``_near_idx``,
        ``_near_offsets``) - used to pin the plan against the reference."""
        starts = source_tree.leaf_starts[self.leaves]
        counts = source_tree.leaf_counts[self.leaves]
        csum = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        offs = csum[self.offsets]
        rows = np.repeat(starts - csum[:-1], counts) + np.arange(int(csum[-1]))
        return rows.astype(np.int64), offs


def near_field_plan(source_tree: Octree, target_tree: Octree) -> NearFieldPlan:
    depth = target_tree.depth
    tl = target_tree.leaves
    anchors, _ = decode_codes(tl)
    n = 1 << depth
    offs = np.array(halo_offsets(), dtype=np.int64)
    cand = anchors[:, None, :] + offs[None, :, :]
    inside = np.all((cand >= 0) & (cand < n), axis=2)
    codes = encode_anchors(np.where(inside[..., None], cand, 0).reshape(-1, 3), depth)
    codes = codes.reshape(tl.shape[0], 26)
    codes = np.where(inside, codes, np.iinfo(np.uint64).max)
    codes.sort(axis=1)
    allc = np.concatenate([tl[:, None], codes], axis=1)
    rows = source_tree.lookup(allc.ravel(), depth).reshape(tl.shape[0], 27)
    valid = rows >= 0
    counts = valid.sum(axis=1)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    leaves = rows[valid].astype(np.int64)
    src_counts = np.where(valid, source_tree.leaf_counts[np.maximum(rows, 0)], 0).sum(axis=1)
    n_pairs = int((src_counts * target_tree.leaf_counts).sum())
    return NearFieldPlan(offsets, leaves, n_pairs)


def child_table(tree: Octree, level: int) -> np.ndarray:
    """(n_boxes(level-1), 8) row of each child at ``level`` or -1."""
    kids = tree.level_keys(level)
    prow = np.searchsorted(tree.level_keys(level - 1), parent_codes(kids))
    tab = np.full((tree.level_keys(level - 1).shape[0], 8), -1, dtype=np.int64)
    tab[prow, child_index_codes(kids)] = np.arange(kids.shape[0])
    return tab


def leaf_centers(tree: Octree) -> np.ndarray:
    """float64 leaf centres, same arithmetic as reference ``engine.py:149-156``."""
    anchors, _ = decode_codes(tree.leaves)
    side = tree.domain.box_side(tree.depth)
    return np.ascontiguousarray(np.asarray(tree.domain.origin, dtype=np.float64)
                                + (anchors + 0.5) * side)


@dataclass
class FmmInstance:
    config: FmmConfig
    domain: Domain
    source_tree: Octree
    target_tree: Octree
    expansions: ExpansionOperators
    blas_ops: m2l_blas.M2lBlasOperators | None = None
    buckets: dict = field(default_factory=dict)
    blas_plans: dict = field(default_factory=dict)
    fft_ops: m2l_fft.M2lFftOperators | None = None
    halo_plans: dict = field(default_factory=dict)
    near: NearFieldPlan | None = None
    _timings: dict = field(default_factory=dict, repr=False)
    setup_seconds: float = 0.0
    m2l_calls: list = field(default_factory=list)
    n_near_pairs: int = 0
    _last_charges: np.ndarray | None = None
    _device: object = None
    # sources and targets are one point set (the mutual near field applies)
    self_interaction: bool = False
    # profile=True: an eager, un-graphed evaluate with a CUDA event between
    # every phase (sequential phase times) instead of the graph's own events
    profile: bool = False

    def evaluate(self, charges, gradient=False):
        return evaluate(self, charges, gradient)

    @property
    def timings(self) -> dict:
        """Seconds per operator class of the last evaluate (the reference's
        six timers, engine.py:289-399).  Filled on every evaluate from CUDA
        events recorded inside the evaluate's graph, read on first access."""
        if callable(self._timings):
            self._timings = self._timings()
        return self._timings

    @timings.setter
    def timings(self, value):
        self._timings = value

    def attach_charges(self, charges):
        return evaluate(self, charges)

    def relative_error(self, potentials, leaf=None) -> ErrorStats:
        return relative_error(self, potentials, leaf)

    def operator_timings(self) -> dict:
        return operator_timings(self)

    @property
    def device(self):
        """Device-resident state (built on first use; needs a CUDA device)."""
        if self._device is None:
            from .device import DeviceFmm
            self._device = DeviceFmm(self)
        return self._device


class LazyBuckets(dict):
    """The reference's per-level ``TransferBuckets`` (``m2l_blas.py:214-258``),
    built on first access: the device path needs only the target-stationary
    plans, the level drop-in ``apply_level`` and the tests need the buckets."""

    def __init__(self, source_tree, target_tree, levels):
        super().__init__()
        self._trees = (source_tree, target_tree)
        self._levels = list(levels)

    def __missing__(self, lvl):
        if lvl not in self._levels:
            raise KeyError(lvl)
        b = m2l_blas.bucket_level(*self._trees, lvl)
        self[lvl] = b
        return b

    def _fill(self):
        for lvl in self._levels:
            self[lvl]

    def items(self):
        self._fill()
        return super().items()

    def keys(self):
        return list(self._levels)

    def values(self):
        self._fill()
        return super().values()

    def __iter__(self):
        return iter(self._levels)

    def __len__(self):
        return len(self._levels)

    def __contains__(self, lvl):
        return lvl in self._levels


def _device_build_available() -> bool:
    import os
    if os.environ.get("KIFMM_DEVICE_SETUP", "1") == "0":
        return False
    try:
        import torch
        from . import _native
        return torch.cuda.is_available() and os.path.exists(_native.LIB_PATH)
    except Exception:
        return False


def setup(sources, targets, config: FmmConfig, device_build=None) -> FmmInstance:
    """Reference ``engine.setup`` (``engine.py:160``).  ``device_build``
    (default: when a GPU and the library are present) builds the trees, the
    near-field plan and the BLAS-M2L plans on the device (device_setup.py,
    bit-identical to the host build); the reference's bucket lists are then
    built lazily, on first access.  The operators are precomputed on the
    host, bit-identical to the reference (a cuSOLVER version measured slower
    on the B200 box: p = 10, 35 s vs 15 s; see DESIGN.md row f4)."""
    t0 = time.perf_counter()
    config.validate()
    src = np.ascontiguousarray(np.asarray(sources, dtype=np.float64).reshape(-1, 3))
    tgt = np.ascontiguousarray(np.asarray(targets, dtype=np.float64).reshape(-1, 3))
    if src.shape[0] < 1 or tgt.shape[0] < 1:
        raise ConfigError("both point sets must be nonempty")
    domain = Domain.from_points(np.vstack([src, tgt]))
    if device_build is None:
        device_build = _device_build_available()
    if device_build:
        from . import device_setup
        stree = device_setup.octree(src, config.depth, domain)
        ttree = device_setup.octree(tgt, config.depth, domain)
    else:
        stree = Octree(src, config.depth, domain)
        ttree = Octree(tgt, config.depth, domain)
    dt = config.dtype
    exp = ExpansionOperators(config.order_equiv, config.resolved_order_check(), dtype=dt,
                             alpha=config.alpha, cutoff=config.svd_cutoff,
                             inner_scale=config.inner_scale, outer_scale=config.outer_scale)
    inst = FmmInstance(config=config, domain=domain, source_tree=stree, target_tree=ttree,
                       expansions=exp)
    inst.self_interaction = bool(src.shape == tgt.shape and np.array_equal(src, tgt))
    if config.backend == "blas":
        inst.blas_ops = m2l_blas.precompute(
            config.order_equiv, config.resolved_order_check(), sigma_min=config.sigma_min,
            rank_estimate=config.rank_estimate, oversamples=config.oversamples,
            seed=config.seed, dtype=dt, inner_scale=config.inner_scale,
            level_scale=1.0 / domain.box_side(config.depth))
        if device_build:
            inst.buckets = LazyBuckets(stree, ttree, range(2, config.depth + 1))
            for lvl in range(2, config.depth + 1):
                inst.blas_plans[lvl] = device_setup.blas_level_plan(stree, ttree, lvl)
        else:
            for lvl in range(2, config.depth + 1):
                b = m2l_blas.bucket_level(stree, ttree, lvl)
                inst.buckets[lvl] = b
                inst.blas_plans[lvl] = m2l_blas.level_plan_from_buckets(
                    b, ttree.level_keys(lvl).shape[0], child_index_codes(ttree.level_keys(lvl)))
    else:
        inst.fft_ops = m2l_fft.precompute_fft_operators(
            config.order_equiv, dtype=dt, inner_scale=config.inner_scale, workers=config.threads)
        for lvl in range(2, config.depth + 1):
            inst.halo_plans[lvl] = m2l_fft.build_halo_plan(stree, ttree, lvl)
    inst.near = (device_setup.near_field_plan(stree, ttree) if device_build
                 else near_field_plan(stree, ttree))
    inst.n_near_pairs = inst.near.n_pairs
    inst.setup_seconds = time.perf_counter() - t0
    return inst


def as_charge_matrix(charges, n_sources: int) -> np.ndarray:
    """(n,), (n, n_rhs) or flat per-RHS blocks -> (n, n_rhs) (reference kernel.py:54-71)."""
    q = np.asarray(charges)
    if q.ndim == 1:
        if q.shape[0] == n_sources:
            return q.reshape(n_sources, 1)
        if n_sources and q.shape[0] % n_sources == 0:
            return q.reshape(-1, n_sources).T
        raise ValueError(f"charge vector length {q.shape[0]} does not cover {n_sources} sources")
    if q.ndim == 2 and q.shape[0] == n_sources:
        return q
    raise ValueError(f"charge array shape {q.shape} does not match {n_sources} sources")


def evaluate(inst: FmmInstance, charges, gradient=False):
    """Potentials at every target (caller order) for one or more charge
    columns; the whole evaluate runs on the GPU.

    ``gradient=True`` (an extension: the reference is potential-only,
    BASELINE config 3 asks for both) returns ``(potentials, gradients)``
    with ``gradients.shape == potentials.shape + (3,)``: the gradient of the
    potential at each target, from the same local expansions (L2P) and near
    field (P2P)."""
    q_in = np.asarray(charges)
    q = np.ascontiguousarray(as_charge_matrix(q_in, inst.source_tree.n_points), dtype=np.float64)
    inst._last_charges = q
    res = inst.device.evaluate_host(q, timings=inst.profile, gradient=gradient)
    out, grad = res if gradient else (res, None)
    inst.timings = (dict(inst.device.last_timings) if inst.profile
                    else inst.device.graph_timings(q.shape[1], gradient))
    inst.m2l_calls = list(inst.device.last_m2l_calls)
    if q_in.ndim == 1 and q.shape[1] == 1:
        out = out[:, 0]
        grad = grad[:, 0] if grad is not None else None
    return (out, grad) if gradient else out


def relative_error(inst: FmmInstance, potentials, leaf=None) -> ErrorStats:
    """Mean relative error over one target leaf against the full direct sum
    in float64 (reference ``engine.py:412-451``); the direct sum runs on the
    GPU through the kernel-level boundary."""
    from . import hotloops
    tt = inst.target_tree
    if inst._last_charges is None:
        raise RuntimeError("evaluate must run before relative_error")
    if leaf is None:
        code = tt.leaves[int(np.argmax(tt.leaf_counts))]
    else:
        code = leaf.code if isinstance(leaf, MortonKey) else int(leaf)
    sl = tt.leaf_slice(code)
    rows_tree = np.arange(sl.start, sl.stop)
    rows_orig = tt.perm[rows_tree]
    st = inst.source_tree
    q_tree = np.ascontiguousarray(inst._last_charges[st.perm], dtype=np.float64)
    ref = np.zeros((rows_tree.shape[0], q_tree.shape[1]))
    hotloops.laplace_potentials(np.ascontiguousarray(tt.x[rows_tree]),
                                np.ascontiguousarray(tt.y[rows_tree]),
                                np.ascontiguousarray(tt.z[rows_tree]), st.x, st.y, st.z,
                                q_tree, ref)
    pot = np.asarray(potentials, dtype=np.float64).reshape(tt.n_points, -1)[rows_orig]
    nz = ref != 0
    n_excl = int(ref.size - np.count_nonzero(nz))
    rel = np.zeros_like(ref)
    rel[nz] = np.abs(pot[nz] - ref[nz]) / np.abs(ref[nz])
    per = [rel[nz[:, r], r].mean() if nz[:, r].any() else 0.0 for r in range(ref.shape[1])]
    return ErrorStats(float(max(per)), n_excl)


def operator_timings(inst: FmmInstance) -> dict:
    out = {k: inst.timings.get(k, 0.0) for k in OPERATOR_NAMES}
    out["setup"] = inst.setup_seconds
    return out


def leaf_surface_base(order: int, side: float, scale: float) -> np.ndarray:
    """Unit offsets of a leaf surface (float64), as reference ``engine.py:154``."""
    return surface(order, np.zeros(3), side, scale, np.float64)
