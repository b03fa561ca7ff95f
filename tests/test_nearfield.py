"""Host logic of the near-field plans (CPU): the mutual slot layout
(csrc/p2p_mutual.cu) and the float32 cross-leaf coincidence check."""

import numpy as np
import pytest

from conftest import uniform_points


def _trees(pts, depth):
    from paper_2408_07436_b200.engine import near_field_plan
    from paper_2408_07436_b200.octree import Domain, Octree
    dom = Domain.from_points(pts)
    st = Octree(pts, depth, dom)
    tt = Octree(pts, depth, dom)
    return st, tt, near_field_plan(st, tt)


@pytest.mark.parametrize("n,depth,cube", [(3000, 3, False), (20000, 4, False), (4000, 4, True)])
def test_mutual_slots_partition_every_pair_once(n, depth, cube):
    from paper_2408_07436_b200.nearfield import mutual_slots
    pts = uniform_points(n, seed=4)
    if cube:
        pts = pts ** 3                     # clustered: empty boxes, ragged near lists
    st, tt, near = _trees(pts, depth)
    ms = mutual_slots(near.offsets, near.leaves, st.leaf_counts)
    counts = st.leaf_counts.astype(np.int64)
    assert ms.total == int((counts * (1 + ms.nlow)).sum())
    seen = {}
    for a in range(counts.shape[0]):
        lst = near.leaves[near.offsets[a]:near.offsets[a + 1]]
        assert lst[0] == a and np.all(np.diff(lst[1:]) > 0)
        for e in range(near.offsets[a], near.offsets[a + 1]):
            b = int(near.leaves[e])
            if b > a:
                rel = int(ms.near_dst[e]) - int(ms.base[b])
                assert rel % counts[b] == 0
                slot = rel // counts[b]
                assert 1 <= slot <= ms.nlow[b]
                # the slot is A's position in B's near list
                assert near.leaves[near.offsets[b] + slot] == a
                assert (b, slot) not in seen
                seen[(b, slot)] = a
            else:
                assert ms.near_dst[e] == -1
    for b in range(counts.shape[0]):
        assert sorted(s for (bb, s) in seen if bb == b) == list(range(1, ms.nlow[b] + 1))


def test_mutual_decomposition_reproduces_the_near_field():
    """Row sums (self + upper pairs) in slot 0 and column sums of the lower
    pairs in slots 1..nlow add up to the reference's per-target-leaf P2P
    (engine.py:224-256 + _hot.pyx:91-138), float64 emulation."""
    from paper_2408_07436_b200.nearfield import mutual_slots
    pts = uniform_points(2500, seed=6)
    st, tt, near = _trees(pts, 3)
    q = np.random.default_rng(7).random(st.n_points)
    P = np.full(mutual_slots(near.offsets, near.leaves, st.leaf_counts).total, np.nan)
    ms = mutual_slots(near.offsets, near.leaves, st.leaf_counts)
    xyz = np.stack([st.x, st.y, st.z], axis=1)
    start, cnt = st.leaf_starts, st.leaf_counts

    def kmat(a, b):
        d = xyz[start[a]:start[a] + cnt[a], None, :] - xyz[None, start[b]:start[b] + cnt[b], :]
        r = np.sqrt((d ** 2).sum(-1))
        with np.errstate(divide="ignore"):
            return np.where(r > 0, 1.0 / r, 0.0)

    for a in range(cnt.shape[0]):
        row = kmat(a, a) @ q[start[a]:start[a] + cnt[a]]
        for e in range(near.offsets[a] + 1, near.offsets[a + 1]):
            b = int(near.leaves[e])
            if b < a:
                continue
            k = kmat(a, b)
            row += k @ q[start[b]:start[b] + cnt[b]]
            d = ms.near_dst[e]
            P[d:d + cnt[b]] = k.T @ q[start[a]:start[a] + cnt[a]]
        P[ms.base[a]:ms.base[a] + cnt[a]] = row
    got = np.zeros(st.n_points)
    for b in range(cnt.shape[0]):
        for s in range(1 + ms.nlow[b]):
            got[start[b]:start[b] + cnt[b]] += P[ms.base[b] + s * cnt[b]:
                                                 ms.base[b] + (s + 1) * cnt[b]]
    assert not np.isnan(P).any()
    # direct: each target leaf against its gathered near sources
    want = np.zeros(st.n_points)
    for b in range(cnt.shape[0]):
        for e in range(near.offsets[b], near.offsets[b + 1]):
            s_ = int(near.leaves[e])
            want[start[b]:start[b] + cnt[b]] += kmat(b, s_) @ q[start[s_]:start[s_] + cnt[s_]]
    assert np.allclose(got, want, rtol=1e-12, atol=0)


def test_mutual_slots_reject_asymmetric_lists():
    from paper_2408_07436_b200.nearfield import mutual_slots
    # leaf 0 lists 1 as a neighbour, leaf 1 does not list 0
    with pytest.raises(ValueError):
        mutual_slots(np.array([0, 2, 3]), np.array([0, 1, 1]), np.array([2, 3]))


def test_f32_cross_leaf_coincidence():
    from paper_2408_07436_b200.nearfield import f32_cross_leaf_coincident
    from paper_2408_07436_b200.octree import Domain, Octree
    pts = uniform_points(5000, seed=9)
    dom = Domain.from_points(np.vstack([pts, [[0.0, 0.0, 0.0], [1.0, 1.0, 1.0]]]))
    t = Octree(pts, 3, dom)
    assert not f32_cross_leaf_coincident(t, t)
    # a pair straddling a leaf boundary 0.5 that rounds to one float32 point
    eps = 1e-12
    pair = np.array([[0.5 - eps, 0.3, 0.3], [0.5 + eps, 0.3, 0.3]])
    assert np.float32(pair[0, 0]) == np.float32(pair[1, 0])
    t2 = Octree(np.vstack([pts, pair]), 3, dom)
    assert f32_cross_leaf_coincident(t2, t2)
    # the same coincidence inside one leaf is not a cross-leaf one
    pair_in = np.array([[0.3 - eps, 0.3, 0.3], [0.3 + eps, 0.3, 0.3]])
    t3 = Octree(np.vstack([pts, pair_in]), 3, dom)
    assert not f32_cross_leaf_coincident(t3, t3)
    # separate clouds: a target equal (in float32) to a source of another leaf
    src = Octree(np.vstack([pts, pair[1:]]), 3, dom)
    tgt = Octree(np.vstack([uniform_points(100, seed=1), pair[:1]]), 3, dom)
    assert f32_cross_leaf_coincident(tgt, src)


@pytest.mark.parametrize("case", ["c1", "c2"])
def test_near_plan_digest_matches_reference_loop(case):
    """The vectorised near-field plan (also what oracle/ref_bridge.py gives
    the reference instance) equals the reference's own per-leaf loop
    (engine.py:224-256) at config-1 and config-2 size: digests of the
    reference's _near_idx / _near_offsets recorded by
    tests/golden/make_near_digest.py (unmodified reference setup, 1M points)."""
    import hashlib
    import json
    import os
    from conftest import GOLDEN
    from paper_2408_07436_b200.engine import near_field_plan
    from paper_2408_07436_b200.octree import Domain, Octree
    with open(os.path.join(GOLDEN, "near_digest.json")) as f:
        want = json.load(f)[case]
    pts = np.random.default_rng(want["seed"]).random((want["n_points"], 3))
    dom = Domain.from_points(np.vstack([pts, pts]))
    st = Octree(pts, want["depth"], dom)
    tt = Octree(pts, want["depth"], dom)
    near = near_field_plan(st, tt)
    rows, offs = near.source_rows(st)
    dig = lambda a: hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()
    assert rows.shape[0] == want["near_idx_len"] and offs.shape[0] == want["near_offsets_len"]
    assert near.n_pairs == want["n_near_pairs"]
    assert dig(offs) == want["near_offsets_sha256"]
    assert dig(rows) == want["near_idx_sha256"]
