"""Multi-GPU evaluate: level-2 subtree partition + multipole halo exchange
(SURVEY.md 8(e)).

Partition.  The union of the source and target level-2 boxes is split into
``world`` contiguous Morton runs, balanced by point count.  A rank owns every
box below its level-2 boxes, so at every level its source and target boxes
form one contiguous row range of the (Morton-sorted) level arrays, and P2M,
M2M, L2L, L2P and P2P never cross ranks.

Exchange.  The only cross-rank dependency is M2L: a target's interaction
list reaches sources up to two boxes beyond a parent-aligned boundary (and,
at level 2, almost every box).  Each rank packs the rows of its own
multipoles that other ranks' targets meet and ONE all-gather per group
delivers them (``HaloExchange``): the leaf level right after P2M, on a
communication stream, overlapping the M2M pass; the coarse levels after M2M
(``torch.distributed`` all_gather_into_tensor: NCCL over NVLink/NVSwitch on
GPUs, gloo in the CPU tests).  Charges are an input every rank holds (the
reference API takes the whole charge vector), so the P2P halo needs no
exchange.  Every rank ends with its owned potentials (tree order); one more
all-gather and a row gather give every rank the caller-order result.

Per rank the passes form the same stream DAG as the single-device evaluate
and are captured, collectives included, as one CUDA graph.
``evaluate_local`` runs several ranks' instances in one process (their
generators advanced collective by collective, no kernel ever waits on
another rank), which exercises every device code path of the partitioned
evaluate on a single GPU.
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


# ------------------------------------------------------------ halo exchange
class HaloExchange:
    """Tables of the all-gather halo exchange (host side, numpy).

    Per exchange group (``fine``: the leaf level, sent right after P2M so it
    overlaps the M2M pass; ``coarse``: every level above it, sent after M2M)
    each rank packs the rows of its own multipoles that ANY other rank's
    targets meet - the union of its per-peer send lists - into one buffer,
    padded to the largest rank's size; ONE ``all_gather_into_tensor`` per
    group delivers every rank's buffer to every rank (NVSwitch: the
    all-gather costs one buffer per link whatever the number of peers), and
    a rank moves the rows it needs out of its peers' segments straight into
    its multipole arrays.  ``world x smax`` rows of ``width`` elements."""

    def __init__(self, plans, rank: int, depth: int):
        world = len(plans)
        self.world, self.rank = world, rank
        groups = {"fine": [depth], "coarse": list(range(2, depth))}
        self.groups = {}
        for name, levels in groups.items():
            seg, sizes = {}, []
            for q in range(world):
                off = 0
                for l in levels:
                    rows = [r for r in plans[q].send_rows[l].values() if r.size]
                    u = np.unique(np.concatenate(rows)) if rows else np.zeros(0, np.int64)
                    seg[(q, l)] = (off, u)
                    off += int(u.shape[0])
                sizes.append(off)
            smax = max(max(sizes), 1)
            pack = [(l, seg[(rank, l)][0], seg[(rank, l)][1].astype(np.int32)) for l in levels]
            unpack = []
            for l in levels:
                pos_all, dst_all = [], []
                for q in range(world):
                    if q == rank:
                        continue
                    need = plans[rank].recv_rows[l][q]
                    if not need.size:
                        continue
                    off, u = seg[(q, l)]
                    pos = np.searchsorted(u, need)
                    assert pos.max() < u.shape[0] and np.array_equal(u[pos], need), \
                        "a needed ghost row is missing from its owner's send union"
                    pos_all.append(q * smax + off + pos)
                    dst_all.append(need)
                cat = (lambda a: np.concatenate(a).astype(np.int32) if a else np.zeros(0, np.int32))
                unpack.append((l, cat(pos_all), cat(dst_all)))
            self.groups[name] = dict(levels=levels, smax=smax, pack=pack, unpack=unpack)

    # numpy twins of the device pack / unpack (CPU tests over gloo)
    def pack_host(self, group, mult):
        g = self.groups[group]
        width = int(np.prod(next(iter(mult.values())).shape[1:]))
        dt = next(iter(mult.values())).dtype
        buf = np.zeros((g["smax"], width), dtype=dt)
        for l, off, rows in g["pack"]:
            buf[off: off + rows.shape[0]] = mult[l][rows].reshape(rows.shape[0], width)
        return buf

    def unpack_host(self, group, recv, mult):
        for l, pos, dst in self.groups[group]["unpack"]:
            if dst.size:
                mult[l][dst] = recv.reshape(-1, recv.shape[-1])[pos].reshape(
                    dst.shape[0], *mult[l].shape[1:])


class TorchCollectives:
    """torch.distributed all-gather (NCCL over NVLink/NVSwitch on GPUs, gloo
    in the CPU tests); issued on the current stream, capturable in a graph."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group

    def all_gather(self, send, recv):
        self.dist.all_gather_into_tensor(recv, send, group=self.group)


class StubCollectives:
    """Timing stand-in for ONE rank run alone on a GPU (tools/rank_time.py):
    the rank's own buffer is copied into its segment of the gathered buffer
    (a device copy of the same size the rank contributes), the peers'
    segments keep whatever they held.  Results are meaningless; the rank's
    kernels, their row ranges and the stream DAG are the real ones."""

    def __init__(self, rank):
        self.rank = rank

    def all_gather(self, send, recv):
        n = send.numel()
        recv[self.rank * n: (self.rank + 1) * n].copy_(send)


# ----------------------------------------------------------------- exchangers
class TorchExchanger:
    """Grouped point-to-point exchange over a torch.distributed process group
    (the per-peer lists the all-gather tables are derived from; kept for the
    CPU test of the ghost lists)."""

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


# ------------------------------------------------------------ device evaluate
def restrict_tma_plan(plan, lo, hi):
    """Rank copy of a ``device.tma_level_plan``: the class tiles holding an
    owned target row, every other row masked (-1: computed by the tile's MMA
    but never written)."""
    from .device import tile_pairs, to_dev
    h = plan["h"]
    per_class = -(-h // 4) * -(-h // 4) * -(-h // 8)
    tt = plan["tile_targets"].cpu().numpy().reshape(-1, 128)
    own = (tt >= lo) & (tt < hi)
    keep = own.any(axis=1)
    tile_ids = plan["tile_ids"].cpu().numpy()[keep]
    pairs = tile_pairs(tile_ids, per_class)
    return dict(h=h, n_tiles=int(tile_ids.shape[0]), tile_ids=to_dev(tile_ids, np.int32),
                tile_targets=to_dev(np.where(own, tt, -1)[keep].reshape(-1), np.int32),
                src_slot=plan["src_slot"], pairs=to_dev(pairs, np.int32),
                n_pairs=int(pairs.shape[0]))


class DistributedFmm:
    """One rank's share of the device evaluate (see module docstring).

    The rank runs the same DAG as the single-device evaluate
    (``DeviceFmm._evaluate``) on its owned row ranges: P2M and M2M of its
    subtrees, the tensor-memory / TMA / DMMA sweeps over the class tiles of
    its own targets, the folded downward solves, the mutual near field of
    its leaves (plus the lower neighbours across the boundary) and the L2P
    pass, on the same streams, and - over a real process group - captured
    as one CUDA graph including the two all-gathers."""

    def __init__(self, inst, rank_plan: RankPlan, device_fmm=None, all_plans=None):
        import torch

        from .device import DeviceFmm, to_dev, upload_blas_plan, upload_hadamard_tiles
        self.inst = inst
        self.plan = rank_plan
        self.dev = device_fmm if device_fmm is not None else DeviceFmm(inst)
        d = self.dev
        self.torch = torch
        depth = d.depth
        if inst.config.backend == "blas":
            if d.tma:
                self.tma_plan = {l: restrict_tma_plan(d.tma_plan[l], *rank_plan.tgt_ranges[l])
                                 for l in range(2, depth + 1)}
            else:
                self.blas_plan_dev = {l: upload_blas_plan(p)
                                      for l, p in rank_plan.blas_plans.items()}
        else:
            self.fft_sub = {}
            for l, (clo, chi, scl) in rank_plan.fft_clusters.items():
                self.fft_sub[l] = (clo, chi, to_dev(scl, np.int32), int(scl.shape[0]),
                                   upload_hadamard_tiles(inst.halo_plans[l].halo[clo:chi],
                                                         inst.halo_plans[l].src_color,
                                                         inst.halo_plans[l].tgt_color[clo:chi]))
        # halo exchange tables (need every rank's plan: positions in the
        # peers' send unions)
        self.halo = HaloExchange(all_plans, rank_plan.rank, depth) if all_plans else None
        self._halo_dev = {}
        if self.halo is not None:
            for name, g in self.halo.groups.items():
                self._halo_dev[name] = dict(
                    pack=[(l, off, to_dev(rows, np.int32)) for l, off, rows in g["pack"]],
                    unpack=[(l, to_dev(pos, np.int32), to_dev(dst, np.int32))
                            for l, pos, dst in g["unpack"]])
        # owned points (tree order) and the output gather tables
        tt = inst.target_tree
        lo, hi = rank_plan.tgt_ranges[depth]
        self.p_lo = int(tt.leaf_starts[lo]) if hi > lo else 0
        self.p_hi = int(tt.leaf_starts[hi - 1] + tt.leaf_counts[hi - 1]) if hi > lo else 0
        self.out_max = 1
        self.assemble = None
        if all_plans:
            ranges = []
            for p in all_plans:
                a, b_ = p.tgt_ranges[depth]
                ranges.append((int(tt.leaf_starts[a]) if b_ > a else 0,
                               int(tt.leaf_starts[b_ - 1] + tt.leaf_counts[b_ - 1]) if b_ > a else 0))
            self.out_max = max(max(b_ - a for a, b_ in ranges), 1)
            pos = np.zeros(tt.n_points, dtype=np.int64)
            for q, (a, b_) in enumerate(ranges):
                pos[a:b_] = q * self.out_max + np.arange(b_ - a)
            idx = np.zeros(tt.n_points, dtype=np.int64)
            idx[np.asarray(tt.perm)] = pos               # caller row c <- gathered row idx[c]
            self.assemble = to_dev(idx, np.int32)
        # near field of the owned leaves: the mutual pass also runs the lower
        # neighbours across the boundary (their column sums land in our slots)
        self.mut_order = None
        if d.mutual is not None and hi > lo:
            off, lv = np.asarray(inst.near.offsets), np.asarray(inst.near.leaves)
            near_own = lv[off[lo]: off[hi]]
            need = np.union1d(np.arange(lo, hi), near_own[near_own < lo])
            full = d.mutual["order"].cpu().numpy()
            self.mut_order = to_dev(full[np.isin(full, need)], np.int32)
        self.comm_stream = torch.cuda.Stream()
        self._rank_bufs = {}
        self._graphs = {}

    # -- per-nrhs buffers of the rank path
    def _bufs(self, nrhs):
        if nrhs in self._rank_bufs:
            return self._rank_bufs[nrhs]
        torch, d = self.torch, self.dev
        dev = d.sx.device
        width = nrhs * d.n_e
        rb = {}
        if self.halo is not None:
            for name, g in self.halo.groups.items():
                rb["send_" + name] = torch.zeros(g["smax"] * width, dtype=d.T, device=dev)
                rb["recv_" + name] = torch.zeros(self.halo.world * g["smax"] * width, dtype=d.T,
                                                 device=dev)
            rb["recv_out"] = torch.zeros(self.halo.world * self.out_max * nrhs, dtype=d.T,
                                         device=dev)
        for m in d._buffers(nrhs)["mult"]:
            m.zero_()
        rb["send_out"] = torch.zeros(self.out_max * nrhs, dtype=d.T, device=dev)
        rb["final"] = torch.zeros(d.tx.shape[0] * nrhs, dtype=d.T, device=dev)
        if self.inst.config.backend == "blas":
            rb["acc"] = {}
            for l in range(2, d.depth + 1):
                if d.tma:
                    p = self.tma_plan[l]
                    n = d.blas.acc_elems(d.n_tgt[l], nrhs, p["n_tiles"], tma=True,
                                         n_pairs=p["n_pairs"])
                    n = max(n, d.blas.acc_elems(d.n_tgt[l], nrhs, p["n_tiles"]))
                else:
                    n = d.blas.acc_elems(d.n_tgt[l], nrhs, self.blas_plan_dev[l]["n_tiles"])
                rb["acc"][l] = torch.zeros(max(n, 1), dtype=d.T, device=dev)
        self._rank_bufs[nrhs] = rb
        return rb

    def _pack(self, group, nrhs):
        from .device import P, launch, stream_handle
        d = self.dev
        b, rb = d._buffers(nrhs), self._bufs(nrhs)
        width = nrhs * d.n_e
        send = rb["send_" + group]
        for l, off, rows in self._halo_dev[group]["pack"]:
            if rows.numel():
                launch(f"kifmm_gather_rows_{d.sfx}", P(b["mult"][l]), P(rows), int(rows.numel()),
                       width, send.data_ptr() + off * width * send.element_size(),
                       stream_handle())

    def _unpack(self, group, nrhs):
        from .device import P, launch, stream_handle
        d = self.dev
        b, rb = d._buffers(nrhs), self._bufs(nrhs)
        width = nrhs * d.n_e
        for l, pos, dst in self._halo_dev[group]["unpack"]:
            if dst.numel():
                launch(f"kifmm_move_rows_{d.sfx}", P(rb["recv_" + group]), P(pos), P(dst),
                       int(dst.numel()), width, P(b["mult"][l]), stream_handle())

    # -- the rank's evaluate as a generator: it yields at the collectives
    # ("allgather", send, recv) with the stream they belong on current; the
    # driver (TorchCollectives, or the in-process emulation) performs them.
    def evaluate_gen(self, q_dev, nrhs):
        torch = self.torch
        from .device import Linalg, Off, P, dense_rowmap, launch, stream_handle
        d = self.dev
        b, rb = d._buffers(nrhs), self._bufs(nrhs)
        R, depth = nrhs, d.depth
        n_e, n_c, rf = d.n_e, d.n_c, d.r_fold
        la, sfx = d.la, d.sfx
        sr, tr = self.plan.src_ranges, self.plan.tgt_ranges
        caller = torch.cuda.current_stream()
        main, comm, side = d.hi_stream, self.comm_stream, d.side_stream
        main.wait_stream(caller)
        torch.cuda.set_stream(main)
        mult, loc, phi = b["mult"], b["loc"], b["phi"]
        q = b["q"]
        npts = d.sx.shape[0]
        # charges of the whole cloud (the near-field halo reads its neighbours')
        launch(f"kifmm_gather_pack_{sfx}", P(q_dev), P(d.s_perm), P(d.sx), P(d.sy), P(d.sz), npts,
               R, P(q), P(b["src4"]), stream_handle())
        # ---- P2M of the owned leaves
        lo, hi = sr[depth]
        if hi > lo:
            launch(f"kifmm_p2m_check_{sfx}", P(d.sx), P(d.sy), P(d.sz), P(q), R,
                   P(d.s_start) + 4 * lo, P(d.s_count) + 4 * lo, hi - lo,
                   P(d.s_centers) + 24 * lo, P(d.check_base), n_c, P(phi), stream_handle())
            la.chain((hi - lo) * R, phi, n_c, Linalg.solve_stages(d.up_inv, d.side[depth]),
                     Off(mult[depth], lo * R * n_e), n_e)
        # ---- leaf-level ghosts on the communication stream (overlaps M2M)
        if self.halo is not None:
            comm.wait_stream(main)
            torch.cuda.set_stream(comm)
            self._pack("fine", R)
            yield ("allgather", rb["send_fine"], rb["recv_fine"])
            torch.cuda.set_stream(comm)
            self._unpack("fine", R)
            torch.cuda.set_stream(main)
        tlo, thi = tr[depth]
        out_base = rb["send_out"].data_ptr() - self.p_lo * R * rb["send_out"].element_size()
        guard_bit = 8 if d.p2p_guard else 0

        def leaf_launch(parts, stream):
            launch(f"kifmm_leaf_pass_{sfx}", P(d.tx), P(d.ty), P(d.tz), P(d.t_start) + 4 * tlo,
                   P(d.t_count) + 4 * tlo, thi - tlo, P(d.t_centers) + 24 * tlo,
                   P(d.equiv_base), n_e, P(loc[depth]) + tlo * R * n_e * q.element_size(),
                   P(b["src4"]), npts, P(d.s_start), P(d.s_count), P(d.near_off) + 4 * tlo,
                   P(d.near_leaf), R, None, parts | guard_bit, out_base, stream)

        def p2p_pass(stream):
            if thi <= tlo:
                return
            if self.mut_order is not None:
                mut = d.mutual
                launch(f"kifmm_p2p_mutual_{sfx}", P(d.tx), P(d.ty), P(d.tz),
                       int(self.mut_order.numel()), P(b["src4"]), npts, P(d.near_off),
                       P(mut["pack"]), P(self.mut_order), R, mut["total"], int(d.p2p_guard),
                       P(b["pmut"]), stream)
                launch(f"kifmm_p2p_mutual_reduce_{sfx}", P(d.t_start) + 4 * tlo,
                       P(d.t_count) + 4 * tlo, thi - tlo, R, None, P(mut["base"]) + 4 * tlo,
                       P(mut["nlow"]) + 4 * tlo, mut["total"], P(b["pmut"]), out_base, stream)
            else:
                leaf_launch(2, stream)

        def fork_p2p():
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                p2p_pass(side.cuda_stream)

        def m2l(lvl, after_sweep=None):
            """t_l = check_l . U_dn on the owned target rows of the level."""
            lo_, hi_ = tr[lvl]
            n_t = d.n_tgt[lvl]
            t_l = b["t_lv"][lvl]
            scale = 1.0 / d.side[lvl]
            if hi_ <= lo_:
                if after_sweep is not None:
                    after_sweep()
                return
            if self.inst.config.backend == "blas" and d.tma:
                d.blas.run_level_tma(self.tma_plan[lvl], mult[lvl], d.n_src[lvl], n_t, R, scale,
                                     b["qt_lv"][lvl], b["dense"][lvl], rb["acc"][lvl], None,
                                     check=t_l, after_sweep=after_sweep,
                                     rows=(lo_, hi_))
                return
            check = b["phi_lv"][lvl]
            if self.inst.config.backend == "blas":
                d.blas.run_level_rows(self.blas_plan_dev[lvl], mult[lvl], d.n_src[lvl], lo_, hi_,
                                      R, scale, check, b["qt_lv"][lvl], rb["acc"][lvl])
            else:
                self._fft_level(lvl, mult[lvl], R, check)
            if after_sweep is not None:
                after_sweep()
            la.gemm((hi_ - lo_) * R, rf, n_c, 1.0, Off(check, lo_ * R * n_c), n_c, d.dn_u, rf,
                    Off(t_l, lo_ * R * rf), rf)

        def solve_level(lvl):
            lo_, hi_ = tr[lvl]
            if hi_ > lo_:
                la.gemm((hi_ - lo_) * R, n_e, rf, d.side[lvl], Off(b["t_lv"][lvl], lo_ * R * rf),
                        rf, d.dn_vv, n_e, Off(loc[lvl], lo_ * R * n_e), n_e)

        forked = {}

        def fork_m2l(lvl, after_sweep=None, wait=()):
            st = d.level_streams[lvl]
            st.wait_stream(main)
            for w in wait:
                st.wait_stream(w)
            with torch.cuda.stream(st):
                m2l(lvl, after_sweep)
            forked[lvl] = st

        # the leaf level's M2L waits for its ghosts; the near field is
        # released behind its sweep (as in the single-device evaluate)
        if depth >= 3:
            fork_m2l(depth, after_sweep=fork_p2p,
                     wait=(comm,) if self.halo is not None else ())
        # ---- M2M of the owned subtrees
        for lvl in range(depth, 2, -1):
            plo, phi_ = sr[lvl - 1]
            if phi_ > plo:
                la.chain((phi_ - plo) * R, mult[lvl], n_e,
                         [(d.m2mT, 8 * n_e, n_c, None, 1.0)] + Linalg.solve_stages(d.up_inv, 1.0),
                         Off(mult[lvl - 1], plo * R * n_e), n_e,
                         a_child=Off(d.src_child[lvl], 8 * plo), child_w=n_e, a_nrhs=R)
        # ---- ghosts of the coarse levels
        if self.halo is not None and depth > 2:
            self._pack("coarse", R)
            yield ("allgather", rb["send_coarse"], rb["recv_coarse"])
            torch.cuda.set_stream(main)
            self._unpack("coarse", R)
        elif self.halo is not None:
            torch.cuda.set_stream(main)
        if depth < 3:
            if self.halo is not None:
                main.wait_stream(comm)
            fork_p2p()
        for lvl in range(depth - 1, 2, -1):
            fork_m2l(lvl)
        # ---- downward chain on the owned rows
        for lvl in range(2, depth + 1):
            if lvl not in forked:
                m2l(lvl)
            if lvl == 2:
                solve_level(2)
            if lvl < depth:
                if lvl + 1 in forked:
                    main.wait_stream(forked[lvl + 1])
                lo_, hi_ = tr[lvl]
                n_par = hi_ - lo_
                t_c = b["t_lv"][lvl + 1]
                if n_par and R == 1 and d._l2l_children_dense(lvl + 1):
                    la.gemm(n_par, 8 * rf, n_e, 0.5 / d.side[lvl + 1], Off(loc[lvl], lo_ * n_e),
                            n_e, d.l2lU, 8 * rf, Off(t_c, lo_ * 8 * rf), 8 * rf, accumulate=True)
                elif n_par:
                    tmp = la.scratch(3, n_par * R * 8 * rf, d.T, t_c.device)
                    la.gemm(n_par * R, 8 * rf, n_e, 0.5 / d.side[lvl + 1],
                            Off(loc[lvl], lo_ * R * n_e), n_e, d.l2lU, 8 * rf, tmp, 8 * rf)
                    launch(f"kifmm_scatter_add_rows_{sfx}", P(tmp),
                           P(d._l2l_rowmap(lvl + 1, R)) + 4 * lo_ * R * 8, n_par * R * 8, rf,
                           P(t_c), stream_handle())
                solve_level(lvl + 1)
        for st in forked.values():
            main.wait_stream(st)
        main.wait_stream(side)
        if thi > tlo:
            leaf_launch(1 | 4, stream_handle())                      # L2P, accumulate
        # ---- owned slices (tree order) -> every rank, caller order
        if self.halo is not None:
            yield ("allgather", rb["send_out"], rb["recv_out"])
            torch.cuda.set_stream(main)
            launch(f"kifmm_gather_rows_{sfx}", P(rb["recv_out"]), P(self.assemble),
                   d.tx.shape[0], R, P(rb["final"]), stream_handle())
        caller.wait_stream(main)
        torch.cuda.set_stream(caller)

    def evaluate(self, q_dev, nrhs, coll):
        """Eager rank evaluate over ``coll`` (TorchCollectives); returns the
        caller-order potentials (n_tgt, R) on this rank's device."""
        for _, send, recv in self.evaluate_gen(q_dev, nrhs):
            coll.all_gather(send, recv)
        return self._bufs(nrhs)["final"].view(-1, nrhs)

    def graph_for(self, nrhs, coll):
        """The rank evaluate, collectives included, captured as one CUDA
        graph: (graph, static float64 charges, output).  Falls back to None
        when the capture is refused (the eager DAG is used then)."""
        torch = self.torch
        if nrhs in self._graphs:
            return self._graphs[nrhs]
        d = self.dev
        static_q = torch.zeros(d.sx.shape[0] * nrhs, dtype=torch.float64, device=d.sx.device)
        warm = torch.cuda.Stream()
        warm.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(warm):
            for _ in range(2):
                self.evaluate(static_q, nrhs, coll)
        torch.cuda.current_stream().wait_stream(warm)
        torch.cuda.synchronize()
        import gc
        was = gc.isenabled()
        gc.disable()
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                out = self.evaluate(static_q, nrhs, coll)
            res = (g, static_q, out)
        except Exception as exc:                          # noqa: BLE001 - report, then run eagerly
            import warnings
            warnings.warn(f"rank evaluate: CUDA-graph capture refused ({exc}); running the "
                          f"eager stream DAG")
            torch.cuda.synchronize()
            res = None
        finally:
            if was:
                gc.enable()
        self._graphs[nrhs] = res
        return res

    def evaluate_graphed(self, q_dev, nrhs, coll):
        gr = self.graph_for(nrhs, coll)
        if gr is None:
            return self.evaluate(q_dev, nrhs, coll)
        g, static_q, out = gr
        static_q.copy_(q_dev.reshape(-1))
        g.replay()
        return out

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


# ------------------------------------------------------------ orchestration
def evaluate_local(inst, world: int, charges):
    """All ranks of a ``world``-way partition emulated in one process on the
    current device: every rank's generator is advanced to its next
    collective, the all-gather is emulated by device copies between the
    ranks' buffers, and so on (no kernel ever waits on another rank).
    Returns potentials in the caller's order - must equal the single-device
    evaluate."""
    import torch
    q = np.ascontiguousarray(np.asarray(charges, dtype=np.float64).reshape(inst.source_tree.n_points, -1))
    R = q.shape[1]
    part = make_partition(inst.source_tree, inst.target_tree, world)
    plans = make_rank_plans(inst, part)
    from .device import DeviceFmm
    ranks = [DistributedFmm(inst, p, DeviceFmm(inst), all_plans=plans) for p in plans]
    qd = torch.from_numpy(q).cuda().reshape(-1)
    gens = [r.evaluate_gen(qd, R) for r in ranks]
    base = torch.cuda.current_stream()
    while True:
        reqs = []
        for g in gens:
            torch.cuda.set_stream(base)
            reqs.append(next(g, None))
        torch.cuda.set_stream(base)
        if all(r is None for r in reqs):
            break
        assert all(r is not None for r in reqs), "ranks disagree on the collective sequence"
        torch.cuda.synchronize()
        for _, _, recv in reqs:
            seg = recv.numel() // world
            for q_, (_, send, _) in enumerate(reqs):
                recv[q_ * seg: (q_ + 1) * seg].copy_(send)
        torch.cuda.synchronize()
    torch.cuda.synchronize()
    outs = [r._bufs(R)["final"].view(-1, R).cpu().numpy() for r in ranks]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0]), "ranks assembled different potentials"
    return outs[0]


def rank_sweep_flops(inst, plan: RankPlan, lvl: int) -> float:
    """Algorithmic flop of the rank's share of a level's BLAS-M2L sweep:
    4 k sum_t m_t k_t over the bucket pairs whose target the rank owns
    (SURVEY 8(d))."""
    lo, hi = plan.tgt_ranges[lvl]
    ops = inst.blas_ops
    total = 0.0
    for t, p in enumerate(inst.buckets[lvl].pairs):
        if p is not None:
            total += 4.0 * ops.k * int(((p[1] >= lo) & (p[1] < hi)).sum()) * ops.ranks[t]
    return total


def bench_main(args, bench):
    """torchrun entry for bench.py --gpus N: strong scaling of the same 1M
    points over N ranks (one GPU each).  A step is one partitioned evaluate:
    every rank replays its CUDA graph (its DAG with the two halo all-gathers
    and the result all-gather inside).  Device-timed with CUDA events, L2
    flushed between steps outside the timed region, step time = max over
    ranks; ``e2e`` adds the pinned H2D of the charges on every rank and the
    D2H of the potentials on rank 0."""
    import time

    import torch
    import torch.distributed as dist

    from . import device as D

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        if "MASTER_ADDR" not in os.environ:              # --force-dist without torchrun
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local))
    from . import FmmConfig, setup
    pts, qh = bench.inputs()
    inst = setup(pts, pts, FmmConfig(**bench.CONFIG))
    part = make_partition(inst.source_tree, inst.target_tree, world)
    plans = make_rank_plans(inst, part)
    rk = DistributedFmm(inst, plans[rank], all_plans=plans)
    coll = TorchCollectives()
    q_dev = torch.from_numpy(qh).cuda()
    q_pin = torch.from_numpy(qh).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    R = 1
    graphed = rk.graph_for(R, coll) is not None

    def step():
        return rk.evaluate_graphed(q_dev, R, coll)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    dist.barrier()
    torch.cuda.synchronize()
    with bench.ClockSampler(local) as clk:
        for e0, e1 in ev:
            flush.zero_()                            # evict L2 (not timed)
            e0.record()
            step()
            e1.record()
        torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())

    # per-launch times of one eager pass (every rank takes part in the
    # collectives); the first sweep launched is the leaf level's
    flush.zero_()
    n0 = D.LAUNCH_COUNT[0]
    with D.profile_launches() as prof:
        rk.evaluate(q_dev, R, coll)
    launches = prof.times()
    n_launch = D.LAUNCH_COUNT[0] - n0
    per_kernel = {}
    for name, _, t in launches:
        per_kernel[name.replace("kifmm_", "")] = per_kernel.get(name.replace("kifmm_", ""), 0.0) + t
    sweeps = [(n, t) for n, _, t in launches if "m2l_sweep" in n]

    # e2e: host charges (pinned) -> every rank; potentials -> host on rank 0
    e2e = []
    out = step()
    host = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
    for _ in range(max(args.steps, 10)):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q_dev.copy_(q_pin, non_blocking=True)
        out = step()
        if rank == 0:
            host.copy_(out, non_blocking=True)
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], device="cuda")
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e.append(float(dt.item()))
    e2e_s = float(np.mean(e2e))
    if rank == 0:
        peaks = bench.measured_peaks()
        roof = None
        if inst.config.backend == "blas" and sweeps:
            lvl = inst.config.depth
            algo = rank_sweep_flops(inst, plans[0], lvl)
            peak_tc = peaks["bf16_tflops"] / 2.0 / 3.0
            sweep_ms = sweeps[0][1]
            roof = dict(bound="tensor", kernel=f"{sweeps[0][0]} (level {lvl}, rank 0's tiles)",
                        achieved=algo / (sweep_ms / 1e3) / 1e12, peak=peak_tc, unit="TFLOP/s",
                        frac=algo / (sweep_ms / 1e3) / 1e12 / peak_tc, traffic=None,
                        algorithmic=f"4 k sum_t m_t k_t over rank 0's targets = {algo:.4g} flop",
                        launch_ms=sweep_ms,
                        peak_source="MEASURED_PEAKS.json bf16_tflops / 2 (TF32) / 3 (3xTF32)")
        cpu = None
        if not args.no_cpu_baseline:
            res = bench.cpu_reference_run(pts, qh, steps=1)
            csec = min(res["times"])
            ref = np.asarray(res["potentials"], dtype=np.float64)
            got = host.numpy().astype(np.float64)[:, 0]
            rel = np.abs(got - ref) / np.abs(ref)
            cpu = dict(value=bench.N_POINTS / csec / 1e6, unit="Mpoints/s", cores=res["cores"],
                       kind=res["kind"], sample="one full 1M-point evaluate, all host threads "
                       "(rank 0's process; the other ranks wait)", seconds=csec,
                       parity_max_rel=float(rel.max()), parity_tol=1e-5)
        line = dict(metric=bench.METRIC, value=bench.N_POINTS / (ms / 1e3) / 1e6,
                    unit="Mpoints/s", n_gpus=world, steps=args.steps, warmup=max(args.warmup, 3),
                    ms_per_step=ms, higher_is_better=True, scaling="strong", vs_baseline=None,
                    dtype="f32", data="synthetic (seeded; no dataset involved)",
                    config=dict(bench.workload(), parallelism=f"level-2 subtree partition x{world}",
                                l2="flushed between steps (256 MB write)",
                                execution=("per rank: one CUDA graph (" if graphed else
                                           "per rank: eager stream DAG (graph capture refused; ")
                                          + "P2M, leaf-level halo all-gather overlapping M2M, "
                                          "coarse halo all-gather, sweeps of the owned class "
                                          "tiles, folded downward solves, mutual near field, "
                                          "L2P, all-gather of the owned potentials)"),
                    gpu_launches=n_launch * args.steps, kernel_ms=per_kernel,
                    e2e=dict(value=bench.N_POINTS / e2e_s / 1e6, unit="Mpoints/s",
                             h2d_bytes_per_step=int(qh.nbytes) * world,
                             d2h_bytes_per_step=int(out.numel() * out.element_size())),
                    roofline=roof, cpu_baseline=cpu, clocks=clk.summary())
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0
