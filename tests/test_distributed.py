"""Multi-GPU path, host logic on CPU: partition, ghost plans and the
multipole exchange over a real torch.distributed (gloo, world_size 2/4)
process group, checked against the single-process oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import uniform_points
from oracle import port
from paper_2408_07436_b200 import FmmConfig, setup
from paper_2408_07436_b200.distributed import (HaloExchange, TorchCollectives, TorchExchanger,
                                                make_partition, make_rank_plans,
                                               restrict_buckets)


def _instance(backend, n=6000, depth=4):
    pts = uniform_points(n, seed=31)
    kw = dict(depth=depth, order_equiv=3, backend=backend, precision="f64", sigma_min=1e-8)
    return setup(pts, pts, FmmConfig(**kw))


@pytest.mark.parametrize("world", [2, 3, 8])
def test_partition_is_contiguous_and_complete(world):
    inst = _instance("blas")
    part = make_partition(inst.source_tree, inst.target_tree, world)
    for lvl in range(2, inst.config.depth + 1):
        n_s = inst.source_tree.level_keys(lvl).shape[0]
        n_t = inst.target_tree.level_keys(lvl).shape[0]
        covered_s = np.zeros(n_s, int)
        covered_t = np.zeros(n_t, int)
        for r in range(world):
            lo, hi = part.src_ranges[r][lvl]
            covered_s[lo:hi] += 1
            lo, hi = part.tgt_ranges[r][lvl]
            covered_t[lo:hi] += 1
        assert np.all(covered_s == 1) and np.all(covered_t == 1)
    # a rank's subtrees are closed under parent/child at every level
    for r in range(world):
        for lvl in range(3, inst.config.depth + 1):
            lo, hi = part.src_ranges[r][lvl]
            from paper_2408_07436_b200.octree import parent_codes
            par = parent_codes(inst.source_tree.level_keys(lvl)[lo:hi])
            rows = np.searchsorted(inst.source_tree.level_keys(lvl - 1), par)
            plo, phi = part.src_ranges[r][lvl - 1]
            assert np.all((rows >= plo) & (rows < phi))


@pytest.mark.parametrize("backend", ["blas", "fft"])
def test_ghost_rows_cover_every_m2l_source(backend):
    inst = _instance(backend)
    world = 4
    part = make_partition(inst.source_tree, inst.target_tree, world)
    plans = make_rank_plans(inst, part)
    for p in plans:
        for lvl in range(2, inst.config.depth + 1):
            slo, shi = p.src_ranges[lvl]
            have = set(range(slo, shi))
            for rows in p.recv_rows[lvl].values():
                assert not (set(rows.tolist()) & have)
                have |= set(rows.tolist())
            lo, hi = p.tgt_ranges[lvl]
            if backend == "blas":
                b = restrict_buckets(inst.buckets[lvl], lo, hi)
                need = set(np.concatenate([q[0] for q in b.pairs if q is not None] or
                                          [np.zeros(0, int)]).tolist())
            else:
                plan = inst.halo_plans[lvl]
                cl = np.unique(plan.tgt_slot[lo:hi] // 8) if hi > lo else np.zeros(0, int)
                h = plan.halo[cl]
                scl = set(h[h >= 0].tolist())
                need = {b for b, s in enumerate(plan.src_slot) if s // 8 in scl}
            assert need <= have, (p.rank, lvl, len(need - have))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_rank_plans_tile_only_owned_targets(world):
    """Each rank's BLAS-M2L plan tiles its own target rows only, so the
    per-rank sweep work is its share of the level, and the plans
    together hold every bucket pair of the level exactly once."""
    from paper_2408_07436_b200.m2l_blas import level_plan_from_buckets
    from paper_2408_07436_b200.octree import child_index_codes
    inst = _instance("blas", n=20000, depth=4)
    part = make_partition(inst.source_tree, inst.target_tree, world)
    plans = make_rank_plans(inst, part)
    for lvl in range(2, inst.config.depth + 1):
        tcodes = inst.target_tree.level_keys(lvl)
        full = level_plan_from_buckets(inst.buckets[lvl], tcodes.shape[0],
                                       child_index_codes(tcodes))
        tiles = 0
        pairs = 0
        for p in plans:
            bp = p.blas_plans[lvl]
            lo, hi = p.tgt_ranges[lvl]
            t = bp.tile_targets[bp.tile_targets >= 0]
            assert np.all((t >= lo) & (t < hi))
            assert sorted(t.tolist()) == list(range(lo, hi))
            tiles += bp.tile_class.shape[0]
            pairs += bp.n_pairs
        assert pairs == full.n_pairs
        # ragged class tails per rank add at most 8 tiles per rank
        assert tiles <= full.tile_class.shape[0] + 8 * world


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port_no, backend, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inst = _instance(backend, n=3000, depth=3)
        part = make_partition(inst.source_tree, inst.target_tree, world)
        plan = make_rank_plans(inst, part)[rank]
        q = np.random.default_rng(5).random(inst.source_tree.n_points)
        state = {}
        port.evaluate(inst, q, state=state)          # full oracle state (every rank)
        mult_full = state["multipoles"]
        # this rank only knows its own multipoles ...
        mult = {l: np.full_like(mult_full[l], np.nan) for l in range(2, inst.config.depth + 1)}
        for l in mult:
            lo, hi = plan.src_ranges[l]
            mult[l][lo:hi] = mult_full[l][lo:hi]
        # ... and the exchange brings the ghosts (flat per-peer buffers, all levels)
        levels = sorted(plan.recv_rows)
        sends = {q_: torch.from_numpy(np.concatenate(
            [mult[l][plan.send_rows[l][q_]].ravel() for l in levels])) for q_ in range(world)
            if q_ != rank}
        recvs = {q_: torch.empty(sum(plan.recv_rows[l][q_].shape[0] for l in levels) *
                                 mult_full[2].shape[1] * mult_full[2].shape[2],
                                 dtype=torch.float64) for q_ in range(world) if q_ != rank}
        TorchExchanger().exchange(rank, sends, recvs)
        width = mult_full[2].shape[1] * mult_full[2].shape[2]
        for q_, buf in recvs.items():
            flat = buf.numpy()
            off = 0
            for l in levels:
                rows = plan.recv_rows[l][q_]
                mult[l][rows] = flat[off: off + rows.shape[0] * width].reshape(rows.shape[0],
                                                                              *mult[l].shape[1:])
                off += rows.shape[0] * width
        # the all-gather exchange of the device path (HaloExchange tables):
        # one buffer per group and rank, every rank receives all of them and
        # moves out the rows it needs - must deliver the same ghosts
        plans_all = make_rank_plans(inst, part)
        halo = HaloExchange(plans_all, rank, inst.config.depth)
        mult_ag = {l: np.full_like(mult_full[l], np.nan) for l in mult}
        for l in mult_ag:
            lo, hi = plan.src_ranges[l]
            mult_ag[l][lo:hi] = mult_full[l][lo:hi]
        coll = TorchCollectives()
        for group, g in halo.groups.items():
            if not g["levels"]:
                continue
            send = torch.from_numpy(halo.pack_host(group, mult_ag))
            recv = torch.empty((world * g["smax"], send.shape[1]), dtype=send.dtype)
            coll.all_gather(send, recv)
            halo.unpack_host(group, recv.numpy(), mult_ag)
        for l in levels:
            assert np.array_equal(np.isnan(mult_ag[l]), np.isnan(mult[l])), l
            assert np.array_equal(np.nan_to_num(mult_ag[l]), np.nan_to_num(mult[l])), l
        # every owned target's M2L input is now exact; compare the level checks
        worst = 0.0
        for l in levels:
            lo, hi = plan.tgt_ranges[l]
            side = inst.domain.box_side(l)
            n_t = inst.target_tree.level_keys(l).shape[0]
            if backend == "blas":
                b = restrict_buckets(inst.buckets[l], lo, hi)
                got = port.apply_level(inst.blas_ops, b, np.nan_to_num(mult[l], nan=1e300),
                                       n_t, 1.0 / side)
                want = port.apply_level(inst.blas_ops, inst.buckets[l], mult_full[l], n_t,
                                        1.0 / side)
            else:
                got = port.m2l_fft_level(inst.fft_ops, inst.halo_plans[l],
                                         np.where(np.isnan(mult[l]), 0.0, mult[l]), 1.0 / side)
                want = port.m2l_fft_level(inst.fft_ops, inst.halo_plans[l], mult_full[l],
                                          1.0 / side)
            if hi > lo:
                d = np.abs(got[lo:hi] - want[lo:hi]).max() / np.abs(want).max()
                worst = max(worst, float(d))
        result[rank] = worst
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("backend,world", [("blas", 2), ("fft", 3)])
def test_gloo_exchange_feeds_m2l_exactly(backend, world):
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_rank_main, args=(world, _free_port(), backend, result), nprocs=world, join=True)
    assert len(result) == world
    for r, v in result.items():
        # blas: ghosts carried exactly, the sweep only reads owned+ghost rows
        # (non-ghost rows were poisoned with 1e300); fft: same within rounding
        assert v <= 1e-12, (r, v)
