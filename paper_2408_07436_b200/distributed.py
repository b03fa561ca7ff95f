"""Multi-GPU evaluate: level-2 subtree partition + multipole halo exchange
(SURVEY.md 8(e)).

Partition.  The union of the source and target level-2 boxes is split into
``world`` contiguous Morton runs, balanced by point count.  A rank owns every
box below its level-2 boxes, so at every level its source and target boxes
form one contiguous row range of the (Morton-sorted) level arrays, and P2M,
M2M, L2L, L2P and P2P never cross ranks.

Exchange.  The only cross-rank dependency is M2L: a target's interaction
list reaches sources up to two boxes beyond a parent-aligned boundary (and,
at level 2, almost every box).  After the upward pass each rank packs the
rows of its own multipoles that other ranks' targets meet, and one grouped
point-to-point exchange (``torch.distributed`` batch_isend_irecv: NCCL over
NVLink on GPUs, gloo in the CPU tests) delivers them; the ranks then run the
downward pass on their own targets.  Charges are an input every rank holds
(the reference API takes the whole charge vector), so the P2P halo needs no
exchange.  The result is reduced to rank 0.

``LocalExchanger`` runs several ranks' instances in one process (sequentially,
no kernel ever waits on another rank), which exercises every device code
path of the partitioned evaluate on a single GPU.
"""

from __future__ import annotations

import json
import os
import time
from dataclasses import dataclass, field

import numpy as np

from .m2l_blas import BlasLevelPlan, TransferBuckets, level_plan_from_buckets
from .octree import child_index_codes, decode_codes, encode_anchors, parent_codes


# ------------------------------------------------------------------ partition
def ancestor_codes(codes, level_from: int, level_to: int):
    """Codes of the level-``level_to`` ancestors of level-``level_from`` codes."""
    a, _ = decode_codes(codes)
    return encode_anchors(a >> (level_from - level_to), level_to)


@dataclass
class Partition:
    """Ownership of level-2 subtrees by rank (contiguous Morton runs)."""

    world: int
    l2_codes: np.ndarray          # sorted union of level-2 codes
    l2_owner: np.ndarray          # rank of each code
    src_ranges: list              # [rank][level] -> (lo, hi) rows of the source level array
    tgt_ranges: list              # [rank][level] -> (lo, hi) rows of the target level array

    def owner_rows(self, tree, level):
        """Owner rank of every box of ``tree`` at ``level`` (>= 2)."""
        anc = ancestor_codes(tree.level_keys(level), level, 2)
        return self.l2_owner[np.searchsorted(self.l2_codes, anc)]


def make_partition(source_tree, target_tree, world: int) -> Partition:
    depth = source_tree.depth
    codes = np.union1d(source_tree.level_keys(2), target_tree.level_keys(2))
    weight = np.zeros(codes.shape[0], dtype=np.float64)
    for tree in (source_tree, target_tree):
        anc = ancestor_codes(tree.leaves, depth, 2)
        np.add.at(weight, np.searchsorted(codes, anc), tree.leaf_counts)
    # contiguous runs with ~equal weight: cut at the cumulative-weight quantiles
    cum = np.cumsum(weight)
    total = cum[-1] if cum.shape[0] else 0.0
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * r / world, side="left")) + 1)
    cuts.append(codes.shape[0])
    cuts = np.maximum.accumulate(np.minimum(np.array(cuts), codes.shape[0]))
    owner = np.zeros(codes.shape[0], dtype=np.int64)
    for r in range(world):
        owner[cuts[r]:cuts[r + 1]] = r
    part = Partition(world, codes, owner, [], [])
    for r in range(world):
        sr, tr = {}, {}
        for lvl in range(2, depth + 1):
            for tree, rng in ((source_tree, sr), (target_tree, tr)):
                own = part.owner_rows(tree, lvl)
                idx = np.flatnonzero(own == r)
                lo = int(idx[0]) if idx.size else int(np.searchsorted(own, r))
                hi = int(idx[-1]) + 1 if idx.size else lo
                assert np.all(own[lo:hi] == r), "ownership must be contiguous"
                rng[lvl] = (lo, hi)
        part.src_ranges.append(sr)
        part.tgt_ranges.append(tr)
    return part


# ----------------------------------------------------------------- rank plans
def restrict_buckets(buckets: TransferBuckets, lo: int, hi: int) -> TransferBuckets:
    pairs = []
    for p in buckets.pairs:
        if p is None:
            pairs.append(None)
            continue
        keep = (p[1] >= lo) & (p[1] < hi)
        pairs.append((p[0][keep], p[1][keep]) if keep.any() else None)
    return TransferBuckets(buckets.level, pairs)


@dataclass
class RankPlan:
    """Host plan of one rank: owned ranges, restricted M2L plans, ghost rows
    and the exchange lists (global source-box rows per level and peer)."""

    rank: int
    world: int
    src_ranges: dict
    tgt_ranges: dict
    blas_plans: dict = field(default_factory=dict)
    fft_clusters: dict = field(default_factory=dict)   # level -> (clo, chi, source cluster list)
    recv_rows: dict = field(default_factory=dict)      # level -> {peer: rows this rank receives}
    send_rows: dict = field(default_factory=dict)      # level -> {peer: rows this rank sends}


def _needed_sources(inst, lvl, lo, hi):
    """Global source rows an owned target range [lo, hi) meets through M2L."""
    if inst.config.backend == "blas":
        b = restrict_buckets(inst.buckets[lvl], lo, hi)
        rows = [p[0] for p in b.pairs if p is not None]
        return (np.unique(np.concatenate(rows)) if rows else np.zeros(0, np.int64)), b
    plan = inst.halo_plans[lvl]
    clo, chi = _target_cluster_range(plan, lo, hi)
    h = plan.halo[clo:chi]
    scl = np.unique(h[h >= 0])
    slot_box = np.full(plan.n_src_clusters * 8, -1, dtype=np.int64)
    slot_box[plan.src_slot] = np.arange(plan.src_slot.shape[0])
    boxes = slot_box[(scl[:, None] * 8 + np.arange(8)[None, :]).ravel()] if scl.size else \
        np.zeros(0, np.int64)
    return np.unique(boxes[boxes >= 0]), (clo, chi, scl)


def _target_cluster_range(plan, lo, hi):
    if hi <= lo:
        return 0, 0
    cl = plan.tgt_slot[lo:hi] // 8
    return int(cl.min()), int(cl.max()) + 1


def make_rank_plans(inst, part: Partition):
    depth = inst.config.depth
    plans = [RankPlan(r, part.world, part.src_ranges[r], part.tgt_ranges[r])
             for r in range(part.world)]
    for lvl in range(2, depth + 1):
        owner = part.owner_rows(inst.source_tree, lvl)
        for p in plans:
            lo, hi = p.tgt_ranges[lvl]
            need, extra = _needed_sources(inst, lvl, lo, hi)
            if inst.config.backend == "blas":
                tcodes = inst.target_tree.level_keys(lvl)
                # tiles of the owned targets only: each rank sweeps its share
                p.blas_plans[lvl] = level_plan_from_buckets(extra, tcodes.shape[0],
                                                            child_index_codes(tcodes),
                                                            owned=(lo, hi))
            else:
                p.fft_clusters[lvl] = extra
            slo, shi = p.src_ranges[lvl]
            ghost = need[(need < slo) | (need >= shi)]
            p.recv_rows[lvl] = {q: ghost[owner[ghost] == q].astype(np.int64)
                                for q in range(part.world) if q != p.rank}
        for p in plans:
            p.send_rows[lvl] = {q.rank: q.recv_rows[lvl][p.rank] for q in plans if q.rank != p.rank}
    return plans


# ----------------------------------------------------------------- exchangers
class TorchExchanger:
    """Grouped point-to-point exchange over a torch.distributed process group
    (NCCL on GPUs, gloo for the CPU tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def exchange(self, rank, sends: dict, recvs: dict):
        """sends/recvs: {peer: tensor}; fills the recv tensors."""
        ops = []
        for peer, t in sends.items():
            if t.numel():
                ops.append(self.dist.P2POp(self.dist.isend, t, peer, group=self.group))
        for peer, t in recvs.items():
            if t.numel():
                ops.append(self.dist.P2POp(self.dist.irecv, t, peer, group=self.group))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()


class LocalExchanger:
    """In-process exchange between emulated ranks (one GPU or CPU): the pack
    buffers of every rank are posted, then copied into the receivers."""

    def __init__(self):
        self.posted = {}

    def post(self, rank, sends):
        self.posted[rank] = sends

    def deliver(self, rank, recvs):
        for peer, t in recvs.items():
            if t.numel():
                t.copy_(self.posted[peer][rank])


# ------------------------------------------------------------ device evaluate
class DistributedFmm:
    """One rank's share of the device evaluate (see module docstring)."""

    def __init__(self, inst, rank_plan: RankPlan, device_fmm=None):
        import torch

        from .device import DeviceFmm, to_dev, upload_blas_plan, upload_hadamard_tiles
        self.inst = inst
        self.plan = rank_plan
        self.dev = device_fmm if device_fmm is not None else DeviceFmm(inst)
        d = self.dev
        self.torch = torch
        R = 1
        self.rows_dev = {}
        for lvl, peers in rank_plan.recv_rows.items():
            for q, rows in peers.items():
                self.rows_dev[("recv", lvl, q)] = to_dev(rows, np.int32)
        for lvl, peers in rank_plan.send_rows.items():
            for q, rows in peers.items():
                self.rows_dev[("send", lvl, q)] = to_dev(rows, np.int32)
        if inst.config.backend == "blas":
            self.blas_plan_dev = {l: upload_blas_plan(p) for l, p in rank_plan.blas_plans.items()}
        else:
            self.fft_sub = {}
            for l, (clo, chi, scl) in rank_plan.fft_clusters.items():
                self.fft_sub[l] = (clo, chi, to_dev(scl, np.int32), int(scl.shape[0]),
                                   upload_hadamard_tiles(inst.halo_plans[l].halo[clo:chi],
                                                         inst.halo_plans[l].src_color,
                                                         inst.halo_plans[l].tgt_color[clo:chi]))
        del R

    def _acc(self, lvl, nrhs):
        """Sweep accumulator of this rank's plan at ``lvl`` (the rank tiles
        only its own targets, so its vector split - and the accumulator
        width - differ from the single-device plan's)."""
        key = (lvl, nrhs)
        if not hasattr(self, "_accs"):
            self._accs = {}
        if key not in self._accs:
            d = self.dev
            n = d.blas.acc_elems(d.n_tgt[lvl], nrhs, self.blas_plan_dev[lvl]["n_tiles"])
            self._accs[key] = self.torch.zeros(max(n, 1), dtype=d.T, device=d.sx.device)
        return self._accs[key]

    # -- exchange buffers: one flat buffer per peer holding all levels' rows
    def _pack_lists(self, kind):
        out = {}
        for q in range(self.plan.world):
            if q == self.plan.rank:
                continue
            out[q] = [(lvl, self.rows_dev[(kind, lvl, q)])
                      for lvl in sorted(self.plan.recv_rows)]
        return out

    def pack(self, nrhs):
        """Send buffers {peer: flat tensor} of this rank's owned multipoles."""
        from .device import P, launch, stream_handle
        d = self.dev
        b = d._buffers(nrhs)
        width = nrhs * d.n_e
        sends = {}
        for q, lst in self._pack_lists("send").items():
            n = sum(int(rows.numel()) for _, rows in lst)
            buf = self.torch.empty(n * width, dtype=d.T, device=d.sx.device)
            off = 0
            for lvl, rows in lst:
                k = int(rows.numel())
                if k:
                    launch(f"kifmm_gather_rows_{d.sfx}", P(b["mult"][lvl]), P(rows), k, width,
                           buf.data_ptr() + off * width * buf.element_size(), stream_handle())
                off += k
            sends[q] = buf
        return sends

    def recv_buffers(self, nrhs):
        d = self.dev
        width = nrhs * d.n_e
        return {q: self.torch.empty(sum(int(r.numel()) for _, r in lst) * width, dtype=d.T,
                                    device=d.sx.device)
                for q, lst in self._pack_lists("recv").items()}

    def unpack(self, recvs, nrhs):
        from .device import P, launch, stream_handle
        d = self.dev
        b = d._buffers(nrhs)
        width = nrhs * d.n_e
        for q, lst in self._pack_lists("recv").items():
            buf = recvs[q]
            off = 0
            for lvl, rows in lst:
                k = int(rows.numel())
                if k:
                    launch(f"kifmm_scatter_rows_{d.sfx}",
                           buf.data_ptr() + off * width * buf.element_size(), P(rows), k, width,
                           P(b["mult"][lvl]), stream_handle())
                off += k

    # -- passes
    def upward(self, q_dev, nrhs):
        """Charge intake, P2M of owned leaves, M2M of owned subtrees."""
        from .device import P, launch, stream_handle
        d = self.dev
        b = d._buffers(nrhs)
        s = stream_handle()
        R, n_e, n_c, depth = nrhs, d.n_e, d.n_c, d.depth
        q = b["q"]
        launch(f"kifmm_gather_charges_{d.sfx}", P(q_dev), P(d.s_perm), d.sx.shape[0], R, P(q), s)
        launch(f"kifmm_pack_sources_{d.sfx}", P(d.sx), P(d.sy), P(d.sz), P(q), d.sx.shape[0], R,
               P(b["src4"]), s)
        isz = q.element_size()
        lo, hi = self.plan.src_ranges[depth]
        nl = hi - lo
        mult, phi, tmp = b["mult"], b["phi"], b["tmp"]
        if nl:
            launch(f"kifmm_p2m_check_{d.sfx}", P(d.sx), P(d.sy), P(d.sz), P(q), R,
                   P(d.s_start) + 4 * lo, P(d.s_count) + 4 * lo, nl, P(d.s_centers) + 24 * lo,
                   P(d.check_base), n_c, P(phi), s)
            d.la.solve(d.up_inv, phi, nl * R, _View(mult[depth], lo * R * n_e, isz), d.side[depth],
                       tmp)
        for lvl in range(depth, 2, -1):
            plo, phi_ = self.plan.src_ranges[lvl - 1]
            n_par = phi_ - plo
            if not n_par:
                continue
            st = b["stack"]
            launch(f"kifmm_stack_children_{d.sfx}", P(mult[lvl]), P(d.src_child[lvl]) + 4 * 8 * plo,
                   n_par, R, n_e, P(st), s)
            d.la.gemm(n_par * R, n_c, 8 * n_e, 1.0, st, 8 * n_e, d.m2mT, n_c, phi, n_c)
            d.la.solve(d.up_inv, phi, n_par * R, _View(mult[lvl - 1], plo * R * n_e, isz), 1.0,
                       tmp)

    def downward(self, nrhs):
        """M2L + solve + L2L of owned targets, then the leaf pass; returns the
        (global, caller-order) output buffer with this rank's targets filled
        and every other entry zero."""
        from .device import BlasDevice, P, launch, stream_handle
        d = self.dev
        b = d._buffers(nrhs)
        s = stream_handle()
        R, n_e, n_c, depth = nrhs, d.n_e, d.n_c, d.depth
        mult, phi, tmp, loc = b["mult"], b["phi"], b["tmp"], b["loc"]
        isz = phi.element_size()
        for lvl in range(2, depth + 1):
            loc[lvl].zero_()
        for lvl in range(2, depth + 1):
            lo, hi = self.plan.tgt_ranges[lvl]
            n_t_all = d.n_tgt[lvl]
            check = phi[: n_t_all * R * n_c]
            if hi > lo:
                if self.inst.config.backend == "blas":
                    bd = d.blas
                    plan = self.blas_plan_dev[lvl]
                    bd.run_level_rows(plan, mult[lvl], d.n_src[lvl], lo, hi, R, 1.0 / d.side[lvl],
                                      check, b["qt_lv"][lvl], self._acc(lvl, R))
                else:
                    self._fft_level(lvl, mult[lvl], R, check)
                d.la.solve(d.dn_inv, _View(check, lo * R * n_c, isz), (hi - lo) * R,
                           _View(loc[lvl], lo * R * n_e, isz), d.side[lvl], tmp, accumulate=True)
            if lvl < depth and hi > lo:
                n_par = hi - lo
                d.la.gemm(n_par * R, 8 * n_c, n_e, 1.0, _View(loc[lvl], lo * R * n_e, isz), n_e,
                          d.l2lT, 8 * n_c, phi, 8 * n_c)
                rowmap = d._l2l_rowmap(lvl + 1, R)
                d.la.solve(d.dn_inv, phi, n_par * R * 8, loc[lvl + 1], 0.5, tmp, accumulate=True,
                           rowmap=_View(rowmap, lo * R * 8, 4))
        out = b["out"]
        out.zero_()
        lo, hi = self.plan.tgt_ranges[depth]
        if hi > lo:
            launch(f"kifmm_leaf_pass_{d.sfx}", P(d.tx), P(d.ty), P(d.tz), P(d.t_start) + 4 * lo,
                   P(d.t_count) + 4 * lo, hi - lo, P(d.t_centers) + 24 * lo, P(d.equiv_base), n_e,
                   P(loc[depth]) + lo * R * n_e * isz, P(b["src4"]), d.sx.shape[0],
                   P(d.s_start), P(d.s_count), P(d.near_off) + 4 * lo, P(d.near_leaf), R,
                   P(d.t_perm), 3, P(out), s)
        return out[: d.tx.shape[0] * R]

    def _fft_level(self, lvl, mult, nrhs, check):
        from .device import P, hadamard_tiled, launch, stream_handle
        d = self.dev
        b = d._buffers(nrhs)
        plan = d.fft_plan_dev[lvl]
        clo, chi, scl, n_scl, tiles = self.fft_sub[lvl]
        nsc = plan["nsc"]
        n_sub = chi - clo
        qhat = b["qhat_lv"][lvl][: 2 * d.n_freq * nsc * 8 * nrhs]
        phat = b["phat_lv"][lvl][: 2 * d.n_freq * n_sub * 8 * nrhs]
        s = stream_handle()
        launch(f"kifmm_fft_forward_{d.sfx}", P(mult), nrhs, d.order, P(plan["sbox"]), nsc, P(scl),
               n_scl, P(qhat), s)
        hadamard_tiled(d.sfx, d.khat, qhat, tiles, d.n_freq, nsc, n_sub, nrhs, phat, s)
        launch(f"kifmm_fft_inverse_{d.sfx}", P(phat), nrhs, d.order, P(plan["tbox"]) + 4 * 8 * clo,
               n_sub, 1.0 / d.side[lvl], P(check), s)


class _View:
    """A raw device pointer offset into a tensor, usable wherever the launch
    helpers expect a tensor (they only call data_ptr())."""

    def __init__(self, t, elems, itemsize):
        self._p = t.data_ptr() + int(elems) * itemsize

    def data_ptr(self):
        return self._p


# ------------------------------------------------------------ orchestration
def evaluate_local(inst, world: int, charges):
    """All ranks of a ``world``-way partition emulated in one process on the
    current device (sequential, LocalExchanger).  Returns potentials in the
    caller's order - must equal the single-device evaluate."""
    import torch
    q = np.ascontiguousarray(np.asarray(charges, dtype=np.float64).reshape(inst.source_tree.n_points, -1))
    R = q.shape[1]
    part = make_partition(inst.source_tree, inst.target_tree, world)
    plans = make_rank_plans(inst, part)
    from .device import DeviceFmm
    shared = None
    ranks = []
    for p in plans:
        dev = DeviceFmm(inst)          # separate buffers per emulated rank
        ranks.append(DistributedFmm(inst, p, dev))
    qd = torch.from_numpy(q).cuda().reshape(-1)
    ex = LocalExchanger()
    for r in ranks:
        r.upward(qd, R)
    for r in ranks:
        ex.post(r.plan.rank, r.pack(R))
    for r in ranks:
        recvs = r.recv_buffers(R)
        ex.deliver(r.plan.rank, recvs)
        r.unpack(recvs, R)
    total = None
    for r in ranks:
        o = r.downward(R).clone()
        total = o if total is None else total + o
    del shared
    return total.view(-1, R).cpu().numpy()


def bench_main(args, bench):
    """torchrun entry for bench.py --gpus N: strong scaling of the same 1M
    points over N ranks (one GPU each).  Each timed step is device-timed
    (CUDA events), L2 flushed between steps outside the timed region, the
    step time is the max over ranks; ``e2e`` adds the pinned H2D of the
    charges on every rank and the D2H of the reduced potentials on rank 0."""
    import time

    import torch
    import torch.distributed as dist

    from . import device as D

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from . import FmmConfig, setup
    pts, qh = bench.inputs()
    inst = setup(pts, pts, FmmConfig(**bench.CONFIG))
    part = make_partition(inst.source_tree, inst.target_tree, world)
    plans = make_rank_plans(inst, part)
    rk = DistributedFmm(inst, plans[rank])
    ex = TorchExchanger()
    q_dev = torch.from_numpy(qh).cuda()
    q_pin = torch.from_numpy(qh).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    R = 1

    def step():
        rk.upward(q_dev, R)
        sends = rk.pack(R)
        recvs = rk.recv_buffers(R)
        ex.exchange(rank, sends, recvs)
        rk.unpack(recvs, R)
        out = rk.downward(R)
        dist.reduce(out, dst=0)
        return out

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    n0 = D.LAUNCH_COUNT[0]
    with bench.ClockSampler(local) as clk:
        for e0, e1 in ev:
            flush.zero_()                            # evict L2 (not timed)
            e0.record()
            step()
            e1.record()
        torch.cuda.synchronize()
    dist.barrier()
    n_launch = D.LAUNCH_COUNT[0] - n0
    ms = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())

    # e2e: host charges (pinned) -> every rank, reduced potentials -> host on rank 0
    e2e = []
    for _ in range(args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q_dev.copy_(q_pin, non_blocking=True)
        out = step()
        if rank == 0:
            out.cpu()
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], device="cuda")
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e.append(float(dt.item()))
    e2e_s = float(np.mean(e2e))
    if rank == 0:
        line = dict(metric=bench.METRIC, value=bench.N_POINTS / (ms / 1e3) / 1e6,
                    unit="Mpoints/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
                    ms_per_step=ms, higher_is_better=True, scaling="strong", vs_baseline=None,
                    dtype="f32", data="synthetic (seeded; no dataset involved)",
                    config=dict(bench.workload(), parallelism=f"level-2 subtree partition x{world}",
                                l2="flushed between steps (256 MB write)",
                                execution="per rank: upward pass, one grouped NCCL multipole "
                                          "exchange, downward pass, reduce to rank 0"),
                    gpu_launches=n_launch,
                    e2e=dict(value=bench.N_POINTS / e2e_s / 1e6, unit="Mpoints/s",
                             h2d_bytes_per_step=int(qh.nbytes) * world,
                             d2h_bytes_per_step=int(out.numel() * out.element_size())),
                    roofline=None, cpu_baseline=None, clocks=clk.summary())
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0
