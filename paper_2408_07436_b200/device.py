"""Device-resident evaluate: uploads the setup plan once, then runs every
pass of ``evaluate`` (reference ``engine.py:270-404``) on the GPU through the
C-ABI of ``libkifmm_b200.so``.

PyTorch is used only for allocations and the stream; all arithmetic is in
our kernels.  There is no CPU path: constructing a :class:`DeviceFmm`
without a CUDA device raises.

Data layout in HBM (n_rhs = R, T = float32 | float64):
  sources / targets   SoA x, y, z (T) in leaf-Morton order, int32 leaf starts/counts
  leaf centres        float64 (n_leaves, 3); surface offsets float64 (n, 3)
  multipoles[l]       (n_src_boxes(l), R, n_equiv) T
  locals[l]           (n_tgt_boxes(l), R, n_equiv) T
  BLAS-M2L            S padded (n_equiv, kin), U^T (k, n_check), transposed dense cores
                      Dt (316, kin, ko_pad), per-level tile plan (int32)
  FFT-M2L             khat (n_freq, 26, 8, 8) complex, per-level slot/halo tables,
                      qhat (n_freq, n_src_clusters, 8, R), phat (n_freq, n_tgt_clusters, 8, R)
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _native as nat
from .engine import child_table, leaf_centers, leaf_surface_base
from .m2l_blas import TILE_TARGETS, dense_cores, level_plan_from_buckets
from .nearfield import f32_cross_leaf_coincident, mutual_order, mutual_slots
from .octree import class_transfer_table

_NP2T = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("kifmm-b200 evaluates on a CUDA device only; none is visible "
                           "(there is no CPU fallback)")
    nat.load()


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


def to_dev(a, dtype=None):
    a = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    return torch.from_numpy(a).to(_dev(), non_blocking=False)


def stream_handle():
    return torch.cuda.current_stream().cuda_stream


def P(t):
    return None if t is None else t.data_ptr()


class Off:
    """A tensor's storage from element ``elems`` on, wherever the launch
    helpers expect a tensor (they only take data_ptr()): the owned row range
    of a rank in the multi-GPU evaluate."""

    def __init__(self, t, elems):
        self._p = t.data_ptr() + int(elems) * t.element_size()

    def data_ptr(self):
        return self._p


# Optional per-launch event profiling (bench.py roofline): when _PROF is a
# list, every launch appends (entry point, tag, start event, end event).
_PROF = None
_TAG = ""


def set_tag(tag: str):
    global _TAG
    _TAG = tag


_TIMELINE = None     # list: (name, tag, stream, end event) per launch, overlap kept


LAUNCH_COUNT = [0]   # kernel launches through the C ABI (bench gpu_launches)


def launch(name, *args):
    LAUNCH_COUNT[0] += 1
    if _PROF is None:
        st = nat.call(name, *args)
        if _TIMELINE is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(torch.cuda.current_stream())
            _TIMELINE.append((name, _TAG, torch.cuda.current_stream().cuda_stream, e))
        return st
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    st = nat.call(name, *args)
    e1.record()
    _PROF.append((name, _TAG, e0, e1))
    return st


class profile_launches:
    """Context manager collecting per-launch CUDA-event times."""

    def __enter__(self):
        global _PROF
        _PROF = []
        self.records = _PROF
        return self

    def __exit__(self, *exc):
        global _PROF
        _PROF = None
        return False

    def times(self):
        """[(entry point, tag, milliseconds)] after a synchronize."""
        torch.cuda.synchronize()
        return [(n, t, a.elapsed_time(b)) for n, t, a, b in self.records]


def blas_geometry(k: int, itemsize: int):
    """(kin, ko_pad, n_slabs) padding of the compressed rank for the SIMT /
    DMMA sweep kernels; mirrors the launch checks in csrc/m2l_blas.cu."""
    if itemsize == 8:                       # DMMA sweep: 16-wide k chunks, slabs of <= 160
        kin = -(-k // 16) * 16
        n_slabs = -(-k // 160)
        kob = -(-(-(-k // n_slabs)) // 16) * 16
        return kin, n_slabs * kob, n_slabs
    vec = 16 // itemsize
    bkmax = 64
    nch = -(-k // bkmax)
    bk = -(-(-(-k // nch)) // vec) * vec
    kin = nch * bk
    n_slabs = -(-k // 128)
    kob = -(-(-(-k // n_slabs)) // 8) * 8
    return kin, n_slabs * kob, n_slabs


class Linalg:
    """Thin typed wrappers around the GEMM / solve entry points."""

    def __init__(self, sfx: str):
        self.sfx = sfx

    def gemm(self, M, N, K, alpha, A, lda, B, ldb, C, ldc, colscale=None, rowmap=None,
             accumulate=False, asum=1, astride=0):
        launch(f"kifmm_gemm_{self.sfx}", M, N, K, float(alpha), P(A), lda, int(asum), astride,
               P(B), ldb, P(colscale), P(C), ldc, P(rowmap), int(bool(accumulate)),
               stream_handle())

    # widest operator (elements) the fused chain kernel handles well; wider
    # chains (p >= 6 in float64) run as tiled GEMM stages instead
    CHAIN_MAX_N = 256
    # row count from which the stages run as separate (throughput) GEMMs
    CHAIN_GEMM_ROWS = 16384

    def chain(self, M, A, lda, stages, C, ldc, rowmap=None, accumulate=False, asum=1,
              astride=0, a_child=None, child_w=0, a_nrhs=1):
        """Fused operator chain (csrc/chain.cu): stages = [(B, K, N, colscale, alpha), ...]."""
        if max(s[2] for s in stages) > self.CHAIN_MAX_N or max(s[1] for s in stages) > 512 \
                or M >= self.CHAIN_GEMM_ROWS:
            return self._chain_gemms(M, A, lda, stages, C, ldc, rowmap, accumulate, asum,
                                     astride, a_child, child_w, a_nrhs)
        st = list(stages) + [(None, 0, 0, None, 1.0)] * (3 - len(stages))
        launch(f"kifmm_chain_{self.sfx}", M, P(A), lda, int(asum), astride, P(a_child),
               child_w, a_nrhs, len(stages), P(st[0][0]), P(st[1][0]), P(st[2][0]),
               st[0][1], st[0][2], st[1][1], st[1][2], st[2][1], st[2][2],
               P(st[0][3]), P(st[1][3]), P(st[2][3]), float(st[0][4]), float(st[1][4]),
               float(st[2][4]), P(C), ldc, P(rowmap), int(bool(accumulate)), stream_handle())

    def _chain_gemms(self, M, A, lda, stages, C, ldc, rowmap, accumulate, asum, astride,
                     a_child, child_w, a_nrhs):
        """Same chain as sequential tiled GEMMs through scratch buffers."""
        T = torch.float32 if self.sfx == "f32" else torch.float64
        dev = torch.device("cuda", torch.cuda.current_device())
        if a_child is not None:
            n_par = M // a_nrhs
            x = self.scratch(0, M * 8 * child_w, T, dev)
            launch(f"kifmm_stack_children_{self.sfx}", P(A), P(a_child), n_par, a_nrhs, child_w,
                   P(x), stream_handle())
            A, lda, asum = x, 8 * child_w, 1
        rows = M
        for i, (B, K, N, cs, al) in enumerate(stages):
            last = i + 1 == len(stages)
            if last:
                self.gemm(rows, N, K, al, A, lda, B, N, C, ldc, colscale=cs, rowmap=rowmap,
                          accumulate=accumulate, asum=asum, astride=astride)
            else:
                y = self.scratch(1 + (i & 1), rows * N, T, dev)
                self.gemm(rows, N, K, al, A, lda, B, N, y, N, colscale=cs, asum=asum,
                          astride=astride)
                rows = rows * N // stages[i + 1][1]
                A, lda, asum, astride = y, stages[i + 1][1], 1, 0

    def rowchain(self, M, A, lda, stages, asum=1, astride=0):
        """Fused float32 row chain for tall inputs (csrc/rowchain.cu): stages =
        [(B, K, N, colscale, alpha, C, ldc, rowmap, accumulate), ...] with an
        optional output C after every stage; dimensions <= 64."""
        st = list(stages) + [(None, 0, 0, None, 1.0, None, 0, None, False)] * (3 - len(stages))
        launch("kifmm_rowchain_f32", M, P(A), lda, int(asum), astride, len(stages),
               P(st[0][0]), P(st[1][0]), P(st[2][0]), st[0][1], st[0][2], st[1][2], st[2][2],
               P(st[0][3]), P(st[1][3]), P(st[2][3]), float(st[0][4]), float(st[1][4]),
               float(st[2][4]), P(st[0][5]), P(st[1][5]), P(st[2][5]), st[0][6], st[1][6],
               st[2][6], P(st[0][7]), P(st[1][7]), P(st[2][7]), int(bool(st[0][8])),
               int(bool(st[1][8])), int(bool(st[2][8])), stream_handle())

    def scratch(self, slot, n, T, dev):
        """Grow-only scratch buffers (allocated outside graph capture on the
        eager warm-up pass, reused afterwards).  A buffer that is outgrown is
        retired, never freed: CUDA graphs captured earlier (another n_rhs)
        keep its raw pointer and must not replay into recycled memory."""
        if not hasattr(self, "_scratch"):
            self._scratch = {}
            self._retired = []
        slot = (torch.cuda.current_stream().cuda_stream, slot, T)   # per stream: levels overlap
        t = self._scratch.get(slot)
        if t is None or t.numel() < n:
            if t is not None:
                self._retired.append(t)
            t = torch.empty(n, dtype=T, device=dev)
            self._scratch[slot] = t
        return t

    @staticmethod
    def solve_stages(inv, scale):
        """The factored pseudo-inverse as two chain stages (expansion.py:78-82):
        (x . U) * inv_vals, then . V^T * scale."""
        u, vals, vt = inv
        n_c, r = u.shape
        return [(u, n_c, r, vals, 1.0), (vt, r, vt.shape[1], None, scale)]

    def solve(self, inv, phi, M, out, scale, tmp, accumulate=False, rowmap=None):
        """out[rowmap] (+)= scale * V diag(inv_vals) U^T phi^T, row form
        (reference expansion.py:78-82 applied through engine._solve_block)."""
        u, vals, vt = inv
        n_c, r = u.shape
        n_e = vt.shape[1]
        self.gemm(M, r, n_c, 1.0, phi, n_c, u, r, tmp, r, colscale=vals)
        self.gemm(M, n_e, r, scale, tmp, r, vt, n_e, out, n_e, rowmap=rowmap,
                  accumulate=accumulate)


SM_COUNT = 148


def sweep_splits(n_tiles: int, n_slabs: int) -> int:
    """Pieces of the 189-vector range per tile so a level fills ~4 CTAs per SM."""
    work = max(1, n_tiles * n_slabs)
    return int(min(63, max(1, -(-4 * SM_COUNT // work))))


def sparse_tile_lists(src: np.ndarray, n_tiles: int):
    """Per tile: uint16 mask of its 8-row groups meeting a source through each
    vector, the ascending list of vectors with any source (int16, -1 padded)
    and its length (the sparse float64 sweep, csrc/m2l_blas.cu)."""
    pres = (src.reshape(n_tiles, TILE_TARGETS // 8, 8, 189) >= 0).any(axis=2)   # (t, 16, 189)
    gmask = (pres.astype(np.uint32) << np.arange(TILE_TARGETS // 8, dtype=np.uint32)[None, :, None]
             ).sum(axis=1).astype(np.uint16)                                    # (t, 189)
    nz = gmask != 0
    order = np.argsort(~nz, axis=1, kind="stable")
    jlist = np.where(np.take_along_axis(nz, order, axis=1), order, -1).astype(np.int16)
    return gmask, jlist, nz.sum(axis=1).astype(np.int32)


def upload_blas_plan(plan):
    n_tiles = plan.tile_class.shape[0]
    src_dev = getattr(plan, "src_dev", None)          # built on the device (device_setup)
    if src_dev is None:
        src_t = plan.src.reshape(n_tiles, TILE_TARGETS, 189).transpose(0, 2, 1)
        src_dev = to_dev(np.ascontiguousarray(src_t), np.int32)
    out = dict(n_tiles=n_tiles, tile_targets=to_dev(plan.tile_targets, np.int32),
               tile_class=to_dev(plan.tile_class, np.int32), src=src_dev)
    if n_tiles:
        gmask, jlist, jcount = sparse_tile_lists(plan.src, n_tiles)
        # the sparse sweep pays off when vectors or row groups go unused
        full = int(jcount.sum()) == 189 * n_tiles and bool((gmask == 0xFFFF).all())
        if not full:
            out.update(gmask=to_dev(gmask.view(np.int16)), jlist=to_dev(jlist),
                       jcount=to_dev(jcount))
    return out


def factored_widths(ranks):
    """Padded rank ktp_t of every transfer vector for the factored float64
    sweep (csrc/m2l_factored.cu) and its width class (ntw, slabs): ktp =
    16 * ntw * slabs, one slab up to 160 columns."""
    k16 = -(-np.asarray(ranks, dtype=np.int64) // 16) * 16
    slabs = np.maximum(1, -(-k16 // 160))
    ntw = -(-(k16 // 16) // slabs)
    ntw = np.where(k16 == 0, 0, ntw)
    return (16 * ntw * slabs).astype(np.int32), ntw.astype(np.int32), slabs.astype(np.int32)


def factored_plan(plan_dev, class_tv, ktp, ntw, slabs):
    """Pair tables of the factored sweep from a target-stationary plan, built
    on the device: every (tile, vector, row) with a source is a pair; the
    pairs of a vector t form its W block (rows padded to 128, ktp_t wide) in
    (tile, vector position, row) order.  Returns None when the W offsets do
    not fit int32 (the dense sweep is used then)."""
    n_tiles = plan_dev["n_tiles"]
    src = plan_dev["src"].reshape(n_tiles, 189, TILE_TARGETS)   # int32 source row or -1
    dev = src.device
    tv = class_tv.to(dev).long()[plan_dev["tile_class"].long()]       # (n_tiles, 189)
    valid = src >= 0
    t_flat = tv[:, :, None].expand(n_tiles, 189, TILE_TARGETS)[valid]
    src_flat = src[valid]
    n_pairs = int(t_flat.numel())
    ktp_d = torch.from_numpy(np.asarray(ktp, np.int64)).to(dev)
    counts = torch.bincount(t_flat, minlength=316)
    rows_pad = (counts + TILE_TARGETS - 1) // TILE_TARGETS * TILE_TARGETS
    w16 = rows_pad * (ktp_d // 2)                            # 16-byte units per block
    wbase16 = torch.cumsum(w16, 0) - w16
    w_elems = int(w16.sum().item()) * 2
    if int(w16.sum().item()) >= 2 ** 31:
        return None
    order = torch.argsort(t_flat, stable=True)
    t_sorted = t_flat[order]
    start = torch.cumsum(counts, 0) - counts
    idx_sorted = torch.arange(n_pairs, device=dev) - start[t_sorted]
    pairidx = torch.empty_like(idx_sorted)
    pairidx[order] = idx_sorted
    woff = torch.full(src.shape, -1, dtype=torch.int32, device=dev)
    woff[valid] = (wbase16[t_flat] + pairidx * (ktp_d[t_flat] // 2)).to(torch.int32)
    rowbase = torch.cumsum(rows_pad, 0) - rows_pad
    rows1 = torch.full((int(rows_pad.sum().item()),), -1, dtype=torch.int32, device=dev)
    rows1[rowbase[t_sorted] + idx_sorted] = src_flat[order]
    nt = (rows_pad // TILE_TARGETS).cpu().numpy()
    tile_t = np.repeat(np.arange(316), nt).astype(np.int32)
    tile_first = (np.concatenate([np.arange(n) for n in nt]) * TILE_TARGETS).astype(np.int32) \
        if tile_t.size else np.zeros(0, np.int32)
    rows1 = rows1.view(-1, TILE_TARGETS)
    classes = []
    for key in sorted({(int(ntw[t]), int(slabs[t])) for t in np.unique(tile_t)}):
        sel = np.flatnonzero((ntw[tile_t] == key[0]) & (slabs[tile_t] == key[1]))
        # launch order: by position along the (Morton-ordered) targets first,
        # vector second, so the CTAs in flight at one time gather the q~ rows
        # of one neighbourhood (L2 hits); vector-major order streams the whole
        # q~ array from HBM once per vector
        frac = (tile_first[sel] // TILE_TARGETS) / np.maximum(nt[tile_t[sel]], 1)
        sel = sel[np.lexsort((tile_t[sel], np.floor(frac * max(n_tiles, 1))))]
        sel_d = torch.from_numpy(sel).to(dev)
        classes.append(dict(ntw=key[0], slabs=key[1], n=int(sel.size),
                            tile_t=to_dev(tile_t[sel]), tile_first=to_dev(tile_first[sel]),
                            rows1=rows1[sel_d].contiguous()))
    return dict(woff=woff, wbase16=wbase16.contiguous(), w_elems=max(w_elems, 2),
                classes=classes, n_pairs=n_pairs, W={})


def tf32_split(x: np.ndarray):
    """Host twin of cvt.rna.tf32.f32: x (float32) -> (hi, lo) with hi, lo
    TF32-representable and x = hi + lo + O(2^-22 |x|)."""
    def rna(v):
        bits = np.ascontiguousarray(v, dtype=np.float32).view(np.uint32)
        return ((bits + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)
    x = np.asarray(x, dtype=np.float32)
    hi = rna(x)
    lo = rna((x - hi).astype(np.float32))
    return hi, lo


def pack_tc_cores(cores: np.ndarray, kin: int, n_out: int, kc_max: int = 32) -> np.ndarray:
    """(316, k, k) float32 cores [out a, in b] -> per vector, per K-chunk, the
    canonical K-major no-swizzle UMMA layout [a/8][b/4][a%8][b%4] the
    tcgen05 sweep copies verbatim into shared memory (csrc/m2l_tc.cu)."""
    nt, k, _ = cores.shape
    d = np.zeros((nt, n_out, kin), dtype=np.float32)
    d[:, :k, :k] = cores
    blocks = []
    for c0 in range(0, kin, kc_max):
        kc = min(kc_max, kin - c0)
        blk = d[:, :, c0:c0 + kc].reshape(nt, n_out // 8, 8, kc // 4, 4).transpose(0, 1, 3, 2, 4)
        blocks.append(blk.reshape(nt, -1))
    return np.ascontiguousarray(np.concatenate(blocks, axis=1))


def pack_tmem_cores(hi: np.ndarray, lo: np.ndarray, kp: int) -> np.ndarray:
    """(316, k, k) TF32 hi/lo cores -> (316, 2 kp kp): per vector [B_hi | B_lo],
    each in the canonical K-major no-swizzle layout with one K chunk of width
    kp, so the hi and lo halves continue each other along N (csrc/m2l_tmem.cu)."""
    return np.ascontiguousarray(np.concatenate(
        [pack_tc_cores(hi, kp, kp, kc_max=kp), pack_tc_cores(lo, kp, kp, kc_max=kp)], axis=1))


def locality_transfer_table() -> np.ndarray:
    """(8, 189) class vector lists (the vectors of class_transfer_table)
    reordered for source-row reuse: grouped by the source sub-lattice, then
    by the sub-lattice shift (x, y, z) with z fastest, so consecutive vectors
    of the tensor-memory sweep read source blocks overlapping in 7 of 8 rows
    (L1 hits).  The order only changes the summation order of the fp32
    accumulator (promoted every 4 vectors)."""
    from .octree import transfer_offsets
    offs = transfer_offsets().astype(np.int64)
    base = class_transfer_table()
    rows = []
    for cls in range(8):
        par = np.array([(cls >> 2) & 1, (cls >> 1) & 1, cls & 1])
        q = par[None, :] + offs[base[cls]]
        sp = ((q[:, 0] & 1) << 2) | ((q[:, 1] & 1) << 1) | (q[:, 2] & 1)
        sh = q >> 1
        key = np.lexsort((sh[:, 2], sh[:, 1], sh[:, 0], sp))
        rows.append(base[cls][key])
    return np.stack(rows)


def tma_level_plan(src_codes, tgt_codes, level):
    """Plan of the TMA-fed tcgen05 sweep (csrc/m2l_tma.cu) for one level:
    class tiles of 4 x 4 x 8 same-parity targets, the target row of every
    tile slot, and the dense sub-lattice slot of every source box."""
    from .octree import decode_codes
    h = 1 << (level - 1)
    tx, ty, tz = -(-h // 4), -(-h // 4), -(-h // 8)
    ta, _ = decode_codes(tgt_codes)
    cls = ((ta[:, 0] & 1) << 2) | ((ta[:, 1] & 1) << 1) | (ta[:, 2] & 1)
    i = ta >> 1
    tile = cls * (tx * ty * tz) + ((i[:, 0] // 4) * ty + i[:, 1] // 4) * tz + i[:, 2] // 8
    row = ((i[:, 0] % 4) * 4 + i[:, 1] % 4) * 8 + i[:, 2] % 8
    tile_ids = np.unique(tile)
    slot = np.searchsorted(tile_ids, tile)
    tile_targets = np.full(tile_ids.shape[0] * 128, -1, dtype=np.int32)
    tile_targets[slot * 128 + row] = np.arange(tgt_codes.shape[0])
    sa, _ = decode_codes(src_codes)
    sp = ((sa[:, 0] & 1) << 2) | ((sa[:, 1] & 1) << 1) | (sa[:, 2] & 1)
    si = sa >> 1
    src_slot = sp * h ** 3 + (si[:, 0] * h + si[:, 1]) * h + si[:, 2]
    pairs = tile_pairs(tile_ids, tx * ty * tz)
    return dict(h=h, n_tiles=int(tile_ids.shape[0]), tile_ids=to_dev(tile_ids, np.int32),
                tile_targets=to_dev(tile_targets, np.int32), src_slot=to_dev(src_slot, np.int32),
                pairs=to_dev(pairs, np.int32), n_pairs=int(pairs.shape[0]))


def dense_rowmap(plan, nrhs):
    """Row map of the projection GEMM into the dense sub-lattice array: row
    (box b, rhs r) -> ((p * R + r) * h^3 + cell), p, cell from src_slot[b]."""
    key = ("dense_rowmap", nrhs)
    if key not in plan:
        h3 = plan["h"] ** 3
        slot = plan["src_slot"].long()
        p, cell = slot // h3, slot % h3
        r = torch.arange(nrhs, device=slot.device)
        rm = (p[:, None] * nrhs + r[None, :]) * h3 + cell[:, None]
        plan[key] = rm.reshape(-1).to(torch.int32).contiguous()
    return plan[key]


def tile_pairs(tile_ids: np.ndarray, per_class: int) -> np.ndarray:
    """(n_pairs, 2) slots of same-class tiles processed by one CTA pair of the
    tensor-memory sweep (consecutive slots of a class; an odd class repeats
    its last slot, both CTAs then write the same rows)."""
    cls = tile_ids // per_class
    out = []
    for c in np.unique(cls):
        sl = np.flatnonzero(cls == c)
        if sl.shape[0] % 2:
            sl = np.append(sl, sl[-1])
        out.append(sl.reshape(-1, 2))
    return np.concatenate(out).astype(np.int32) if out else np.zeros((0, 2), np.int32)


class BlasDevice:
    """Device copies of the compressed M2L operators and the level apply:
    projection q~ = M S, fused target-stationary sweep, expansion
    check = level_scale * acc U^T (reference m2l_blas.py:284-326)."""

    def __init__(self, ops, np_dtype, la, tensor_cores=None):
        import os
        dt = np.dtype(np_dtype)
        self.la, self.sfx = la, la.sfx
        self.k = k = ops.k
        self.n_e, self.n_c = ops.s.shape[0], ops.u.shape[0]
        if tensor_cores is None:
            tensor_cores = True
        # float32: tcgen05 3xTF32 sweep (csrc/m2l_tc.cu); float64: FP64 SIMT sweep.
        # (3 TMEM accumulators of n_out <= 160 columns fit the 512-column TMEM;
        # above 256 columns the kernels run one CTA per SM)
        self.tc = bool(tensor_cores) and dt == np.float32 and -(-k // 16) * 16 <= 160
        if self.tc:
            self.kin = -(-k // 8) * 8
            self.ko_pad = -(-k // 16) * 16
            self.n_slabs = 1
            cores32 = dense_cores(ops, np.float64).astype(np.float32)
            hi, lo = tf32_split(cores32)
            self.Bhi = to_dev(pack_tc_cores(hi, self.kin, self.ko_pad))
            self.Blo = to_dev(pack_tc_cores(lo, self.kin, self.ko_pad))
            s_pad = np.zeros((self.n_e, self.kin), dtype=dt)
            s_pad[:, :k] = ops.s
            self.S = to_dev(s_pad)
            self.UT = to_dev(np.ascontiguousarray(ops.u.T), dt)
            self.class_tv = to_dev(class_transfer_table(), np.int32)
            from .octree import transfer_offsets
            self.offsets = to_dev(transfer_offsets(), np.int8)
            # A operand in tensor memory (csrc/m2l_tmem.cu) for ranks <= 64;
            # KIFMM_F32_SWEEP=tma keeps the shared-memory-staged TMA sweep
            self.tmem = self.kin <= 64 and os.environ.get("KIFMM_F32_SWEEP", "tmem") == "tmem"
            if self.tmem:
                self.Bpair = to_dev(pack_tmem_cores(hi, lo, self.kin))
                self.class_tv_local = to_dev(locality_transfer_table(), np.int32)
            return
        self.kin, self.ko_pad, self.n_slabs = blas_geometry(k, dt.itemsize)
        s_pad = np.zeros((self.n_e, self.kin), dtype=dt)
        s_pad[:, :k] = ops.s
        self.S = to_dev(s_pad)
        self.UT = to_dev(np.ascontiguousarray(ops.u.T), dt)          # (k, n_c)
        cores = dense_cores(ops, np.float64)                          # (316, k, k) [out, in]
        dt_pad = np.zeros((cores.shape[0], self.kin, self.ko_pad), dtype=dt)
        dt_pad[:, :k, :k] = cores.transpose(0, 2, 1)
        self.Dt = to_dev(dt_pad)
        self.class_tv = to_dev(class_transfer_table(), np.int32)
        # Factored float64 sweep (csrc/m2l_factored.cu): (q~ vbar_t) ubar_t^T in
        # two passes, 2 ktp (kin + ko_pad) flop per pair instead of the dense
        # 2 kin ko_pad; used when the padded ranks make it clearly cheaper
        # (KIFMM_F64_SWEEP = auto | dense | factored)
        self.factored = False
        mode = os.environ.get("KIFMM_F64_SWEEP", "auto")
        if dt == np.float64 and mode != "dense":
            ktp, ntw, slabs = factored_widths(ops.ranks)
            live = ktp[ktp > 0]
            cheaper = live.size and live.mean() * (self.kin + self.ko_pad) < \
                0.7 * self.kin * self.ko_pad
            if mode == "factored" or cheaper:
                self.factored = True
                self.ktp, self.f_ntw, self.f_slabs = ktp, ntw, slabs
                voff = np.concatenate([[0], np.cumsum(self.kin * ktp.astype(np.int64))])
                uoff = np.concatenate([[0], np.cumsum(self.ko_pad * ktp.astype(np.int64))])
                vb = np.zeros(max(int(voff[-1]), 1), dtype=np.float64)
                ub = np.zeros(max(int(uoff[-1]), 1), dtype=np.float64)
                for t in range(cores.shape[0]):
                    kt = ops.ubar[t].shape[1]
                    if not kt:
                        continue
                    v = np.zeros((self.kin, ktp[t]))
                    v[:k, :kt] = ops.vbar[t]
                    vb[voff[t]: voff[t + 1]] = v.ravel()
                    u = np.zeros((ktp[t], self.ko_pad))
                    u[:kt, :k] = np.asarray(ops.ubar[t]).T
                    ub[uoff[t]: uoff[t + 1]] = u.ravel()
                self.vbar, self.ubT = to_dev(vb), to_dev(ub)
                self.voff, self.uoff = to_dev(voff[:-1], np.int64), to_dev(uoff[:-1], np.int64)
                self.ktp_dev = to_dev(ktp, np.int32)

    def run_level_rows(self, plan, mult, n_s, lo, hi, nrhs, level_scale, check, qt, acc):
        """Multi-GPU variant for the generic bucket plans (float64, and float32
        ranks above 160): ``plan`` covers only the target rows [lo, hi) (global
        row numbering); the expansion runs on those rows only.  (float32 ranks
        up to 160 take the class-tile plans: run_level_tma with ``rows``.)"""
        la = self.la
        nsplit = sweep_splits(plan["n_tiles"], self.n_slabs)
        ld = nsplit * self.ko_pad
        la.gemm(n_s * nrhs, self.kin, self.n_e, 1.0, mult, self.n_e, self.S, self.kin, qt, self.kin)
        if self.sfx == "f64":
            self.sweep_f64(plan, qt, nrhs, nsplit, acc)
        elif plan["n_tiles"]:
            launch(f"kifmm_m2l_sweep_{self.sfx}", P(qt), P(self.Dt), self.kin, self.ko_pad,
                   P(plan["tile_targets"]), P(plan["tile_class"]), P(plan["src"]),
                   P(self.class_tv), plan["n_tiles"], nrhs, nsplit, P(acc), stream_handle())
        la.gemm((hi - lo) * nrhs, self.n_c, self.k, level_scale, Off(acc, lo * nrhs * ld), ld,
                self.UT, self.n_c, Off(check, lo * nrhs * self.n_c), self.n_c, asum=nsplit,
                astride=self.ko_pad)
        return 3

    def sweep_f64(self, plan, qt, nrhs, nsplit, acc):
        """The float64 bucket sweep of one level plan: factored (compress +
        expand) when the operators call for it, else the dense DMMA sweep
        (sparse variant on plans with unused vectors / row groups)."""
        if not plan["n_tiles"]:
            return
        sparse = "gmask" in plan
        if self.factored:
            if "fact" not in plan:
                plan["fact"] = factored_plan(plan, self.class_tv, self.ktp, self.f_ntw,
                                             self.f_slabs)
            f = plan["fact"]
        else:
            f = None
        if f is not None:
            if nrhs not in f["W"]:
                f["W"][nrhs] = torch.empty(f["w_elems"] * nrhs, dtype=torch.float64,
                                           device=qt.device)
            W = f["W"][nrhs]
            for c in f["classes"]:
                launch("kifmm_m2l_compress_f64", P(qt), self.kin, nrhs, P(self.vbar),
                       P(self.voff), P(self.ktp_dev), P(c["tile_t"]), P(c["tile_first"]),
                       P(c["rows1"]), c["n"], c["ntw"], c["slabs"], P(f["wbase16"]), P(W),
                       f["w_elems"], stream_handle())
            launch("kifmm_m2l_expand_f64", P(W), f["w_elems"], P(self.ubT), P(self.uoff),
                   P(self.ktp_dev), self.ko_pad, P(plan["tile_targets"]), P(plan["tile_class"]),
                   P(f["woff"]), P(self.class_tv), plan["n_tiles"], nrhs, nsplit,
                   P(plan["gmask"]) if sparse else None, P(plan["jlist"]) if sparse else None,
                   P(plan["jcount"]) if sparse else None, P(acc), stream_handle())
        elif sparse:
            launch("kifmm_m2l_sweep_sparse_f64", P(qt), P(self.Dt), self.kin, self.ko_pad,
                   P(plan["tile_targets"]), P(plan["tile_class"]), P(plan["src"]),
                   P(self.class_tv), plan["n_tiles"], nrhs, nsplit, P(plan["gmask"]),
                   P(plan["jlist"]), P(plan["jcount"]), P(acc), stream_handle())
        else:
            launch("kifmm_m2l_sweep_f64", P(qt), P(self.Dt), self.kin, self.ko_pad,
                   P(plan["tile_targets"]), P(plan["tile_class"]), P(plan["src"]),
                   P(self.class_tv), plan["n_tiles"], nrhs, nsplit, P(acc), stream_handle())

    def tmem_splits(self, n_tiles, n_pairs, nrhs):
        """Vector-range split of the persistent tensor-memory sweep (host-side
        query of the library, not a kernel launch)."""
        import ctypes
        out = ctypes.c_int64(0)
        nat.call("kifmm_m2l_sweep_tmem_splits", n_tiles, n_pairs, nrhs, ctypes.addressof(out))
        return int(out.value)

    def run_level_tma(self, plan, mult, n_s, n_t, nrhs, level_scale, qt, dense, acc, solve,
                      check=None, coarse_ctas=0, rows=None, projected=False,
                      after_sweep=None):
        """Engine path for float32: projection -> dense sub-lattice array ->
        tcgen05 sweep (A in tensor memory, or TMA-staged hi/lo planes) ->
        fused epilogue into the locals.

        ``coarse_ctas`` > 0 (a level above the finest in the overlapped
        evaluate): the persistent sweep is confined to about that many CTAs.
        A persistent CTA owns its SM's shared memory, so a coarse level
        spread over all SMs (a few vectors each) keeps the near field off the
        whole machine for its duration; on a few SMs it takes longer but
        runs in the near field's shadow."""
        la = self.la
        if self.tmem:
            nsplit = self.tmem_splits(plan["n_tiles"], plan["n_pairs"], nrhs)
            if coarse_ctas > 0 and plan["n_tiles"] * nrhs <= coarse_ctas:
                nsplit = min(nsplit, max(1, -(-coarse_ctas // (plan["n_tiles"] * nrhs))))
            # projection q~ = M S written straight into the dense parity
            # sub-lattice array (row map (box, rhs) -> plane p*R + r, cell);
            # `projected`: the caller's fused P2M chain has written it already
            if not projected:
                la.gemm(n_s * nrhs, self.kin, self.n_e, 1.0, mult, self.n_e, self.S, self.kin,
                        dense[0], self.kin, rowmap=dense_rowmap(plan, nrhs))
            launch("kifmm_m2l_sweep_tmem_f32", P(dense[0]), P(self.Bpair), self.kin, plan["h"],
                   P(plan["tile_targets"]), P(plan["tile_ids"]), plan["n_tiles"],
                   P(plan["pairs"]), plan["n_pairs"], P(self.class_tv_local), P(self.offsets),
                   nrhs, nsplit, self.ko_pad, P(acc), stream_handle())
        else:
            nsplit = sweep_splits(plan["n_tiles"], 1)
            self._run_tma(plan, mult, n_s, nrhs, qt, dense, acc, nsplit)
        if after_sweep is not None:
            after_sweep()
        if solve is None:
            # t = check . U_dn in one product (acc . (U^T U_dn)); the caller
            # adds the L2L part and applies the rest of the solve
            # (rows: the owned target range of a rank plan)
            r = self.UTU.shape[1]
            lo, hi = rows if rows is not None else (0, n_t)
            ld = nsplit * self.ko_pad
            la.gemm((hi - lo) * nrhs, r, self.k, level_scale, Off(acc, lo * nrhs * ld), ld,
                    self.UTU, r, Off(check, lo * nrhs * r), r, asum=nsplit, astride=self.ko_pad)
            return 3
        inv, side, loc = solve
        la.chain(n_t * nrhs, acc, nsplit * self.ko_pad,
                 [(self.UT, self.k, self.n_c, None, level_scale)]
                 + Linalg.solve_stages(inv, side), loc, inv[2].shape[1], accumulate=True,
                 asum=nsplit, astride=self.ko_pad)
        return 4

    def _run_tma(self, plan, mult, n_s, nrhs, qt, dense, acc, nsplit):
        la = self.la
        la.gemm(n_s * nrhs, self.kin, self.n_e, 1.0, mult, self.n_e, self.S, self.kin, qt, self.kin)
        hi, lo = dense
        # TF32 hi/lo planes split here (splitting raw fp32 q~ in the sweep's
        # shared memory halves the TMA bytes for A but measured slower on
        # B200: the sweep is bound by shared-memory traffic)
        launch("kifmm_dense_split_tf32", P(qt), P(plan["src_slot"]), n_s, nrhs, self.kin,
               plan["h"], P(hi), P(lo), stream_handle())
        launch("kifmm_m2l_sweep_tma_f32", P(hi), P(lo), P(self.Bhi), P(self.Blo), self.kin,
               self.ko_pad, plan["h"], P(plan["tile_targets"]), P(plan["tile_ids"]),
               plan["n_tiles"], P(self.class_tv), P(self.offsets), nrhs, nsplit, P(acc),
               stream_handle())

    def acc_elems(self, n_t, nrhs, n_tiles, tma=False, n_pairs=0):
        ns = sweep_splits(n_tiles, self.n_slabs)
        if tma and self.tmem:
            ns = max(ns, self.tmem_splits(n_tiles, n_pairs, nrhs))
        return n_t * nrhs * ns * self.ko_pad

    def run_level(self, plan, mult, n_s, n_t, nrhs, level_scale, check, qt, acc, solve=None):
        la = self.la
        nsplit = sweep_splits(plan["n_tiles"], self.n_slabs)
        ld = nsplit * self.ko_pad
        la.gemm(n_s * nrhs, self.kin, self.n_e, 1.0, mult, self.n_e, self.S, self.kin, qt, self.kin)
        if self.tc:
            nq = n_s * nrhs * self.kin
            qhi, qlo = qt[nq: 2 * nq], qt[2 * nq: 3 * nq]
            launch("kifmm_split_tf32", P(qt), nq, P(qhi), P(qlo), stream_handle())
            if plan["n_tiles"]:
                launch("kifmm_m2l_sweep_tc_f32", P(qhi), P(qlo), P(self.Bhi), P(self.Blo),
                       self.kin, self.ko_pad, P(plan["tile_targets"]), P(plan["tile_class"]),
                       P(plan["src"]), P(self.class_tv), plan["n_tiles"], nrhs, nsplit, P(acc),
                       stream_handle())
        elif self.sfx == "f64":
            self.sweep_f64(plan, qt, nrhs, nsplit, acc)
        elif plan["n_tiles"]:
            launch(f"kifmm_m2l_sweep_{self.sfx}", P(qt), P(self.Dt), self.kin, self.ko_pad,
                   P(plan["tile_targets"]), P(plan["tile_class"]), P(plan["src"]),
                   P(self.class_tv), plan["n_tiles"], nrhs, nsplit, P(acc), stream_handle())
        if solve is not None:
            # fused M2L epilogue: split-sum . U^T * level_scale, then the
            # check->local solve, accumulated into the locals
            inv, side, loc = solve
            la.chain(n_t * nrhs, acc, ld,
                     [(self.UT, self.k, self.n_c, None, level_scale)]
                     + Linalg.solve_stages(inv, side), loc, inv[2].shape[1], accumulate=True,
                     asum=nsplit, astride=self.ko_pad)
            return 3
        la.gemm(n_t * nrhs, self.n_c, self.k, level_scale, acc, ld, self.UT, self.n_c, check,
                self.n_c, asum=nsplit, astride=self.ko_pad)
        return 3


class DeviceFmm:
    """GPU-resident copy of an :class:`~.engine.FmmInstance` plan."""

    def __init__(self, inst):
        require_cuda()
        self.inst = inst
        cfg = inst.config
        self.cfg = cfg
        self.np_dtype = np.dtype(cfg.dtype)
        self.T = _NP2T[self.np_dtype]
        self.sfx = "f32" if self.np_dtype == np.float32 else "f64"
        self.la = Linalg(self.sfx)
        st, tt = inst.source_tree, inst.target_tree
        exp = inst.expansions
        self.depth = cfg.depth
        self.n_e, self.n_c = exp.n_equiv, exp.n_check
        # near field concurrent with the far field (see evaluate_device)
        self.overlap = os.environ.get("KIFMM_OVERLAP", "1") != "0"
        # persistent CTAs of a coarse level's sweep in the overlapped evaluate
        # (measured: 32; all SMs keeps the near field off the whole machine)
        self.coarse_ctas = 32
        least, greatest = torch.cuda.Stream.priority_range()
        self.side_stream = torch.cuda.Stream(priority=least)
        self.hi_stream = torch.cuda.Stream(priority=greatest)
        mid = max(greatest, least - 1) if least > greatest else least
        self.level_streams = {l: torch.cuda.Stream(priority=mid) for l in range(2, cfg.depth + 1)}
        self.bulk_stream = self.level_streams[cfg.depth]
        dt = self.np_dtype
        leaf_side = inst.domain.box_side(cfg.depth)
        # points
        self.sx, self.sy, self.sz = (to_dev(v, dt) for v in (st.x, st.y, st.z))
        self.tx, self.ty, self.tz = (to_dev(v, dt) for v in (tt.x, tt.y, tt.z))
        self.s_start = to_dev(st.leaf_starts, np.int32)
        self.s_count = to_dev(st.leaf_counts, np.int32)
        self.t_start = to_dev(tt.leaf_starts, np.int32)
        self.t_count = to_dev(tt.leaf_counts, np.int32)
        self.s_perm = to_dev(st.perm, np.int64)
        self.t_perm = to_dev(tt.perm, np.int64)
        self.s_centers = to_dev(leaf_centers(st))
        self.t_centers = to_dev(leaf_centers(tt))
        self.check_base = to_dev(leaf_surface_base(cfg.resolved_order_check(), leaf_side,
                                                   cfg.outer_scale))
        self.equiv_base = to_dev(leaf_surface_base(cfg.order_equiv, leaf_side, cfg.outer_scale))
        if inst.near.offsets.shape[0] > 1 and int(np.diff(inst.near.offsets).max()) > 32:
            raise ValueError("a leaf's near field spans more than 32 leaves (leaf pass limit)")
        self.near_off = to_dev(inst.near.offsets, np.int32)
        self.near_leaf = to_dev(inst.near.leaves, np.int32)
        # float32 rounding can merge points of different leaves: then every
        # near-field pair is guarded against r2 == 0 (reference _hot.pyx:44-50)
        self.p2p_guard = self.sfx == "f32" and f32_cross_leaf_coincident(tt, st)
        # sources == targets (one point set): the mutual near field evaluates
        # each pair of adjacent leaves once (csrc/p2p_mutual.cu); potential
        # path, both precisions (KIFMM_P2P=direct keeps the per-target-leaf pass)
        self.mutual = None
        if (getattr(inst, "self_interaction", False)
                and os.environ.get("KIFMM_P2P", "mutual") == "mutual"
                and np.array_equal(st.perm, tt.perm)):
            ms = mutual_slots(inst.near.offsets, inst.near.leaves, st.leaf_counts)
            self.mutual = dict(base=to_dev(ms.base), nlow=to_dev(ms.nlow), total=ms.total,
                               pack=to_dev(ms.pack(inst.near.offsets, inst.near.leaves,
                                                   st.leaf_starts, st.leaf_counts)),
                               order=to_dev(mutual_order(inst.near.offsets, inst.near.leaves,
                                                         st.leaf_counts)))
        # unit-box operators
        def inv_parts(inv):
            return (to_dev(inv.u, dt), to_dev(inv.inv_vals, dt),
                    to_dev(np.ascontiguousarray(inv.v.T), dt))
        self.up_inv = inv_parts(exp.up_inv)
        self.dn_inv = inv_parts(exp.down_inv)
        self.r_up, self.r_dn = exp.up_inv.rank, exp.down_inv.rank
        self.m2mT = to_dev(np.ascontiguousarray(exp.m2m_kernels.T), dt)
        self.l2lT = to_dev(np.ascontiguousarray(exp.l2l_kernels.T), dt)
        # Folded down-solve operators of the engine's downward pass (float64
        # products, cast once): t = check . U_dn carries each level's M2L and
        # L2L contributions, locals = t . diag(inv) V_dn^T x side.
        u_dn = np.asarray(exp.down_inv.u, dtype=np.float64)               # (n_c, r)
        self.r_fold = u_dn.shape[1]
        self.dn_vv = to_dev(np.asarray(exp.down_inv.inv_vals, np.float64)[:, None]
                            * np.asarray(exp.down_inv.v, np.float64).T, dt)  # (r, n_e)
        l2l = np.asarray(exp.l2l_kernels, dtype=np.float64).T                  # (n_e, 8 n_c)
        n_e_, n_c_ = l2l.shape[0], u_dn.shape[0]
        self.l2lU = to_dev(np.ascontiguousarray(
            (l2l.reshape(n_e_, 8, n_c_) @ u_dn).reshape(n_e_, 8 * self.r_fold)), dt)
        self.dn_u = to_dev(u_dn, dt)
        # tree levels
        self.n_src = [st.level_keys(l).shape[0] for l in range(cfg.depth + 1)]
        self.n_tgt = [tt.level_keys(l).shape[0] for l in range(cfg.depth + 1)]
        self.src_child = {l: to_dev(child_table(st, l), np.int32) for l in range(3, cfg.depth + 1)}
        self._tgt_child_np = {l: child_table(tt, l) for l in range(3, cfg.depth + 1)}
        self._l2l_rowmaps = {}
        self.side = [inst.domain.box_side(l) for l in range(cfg.depth + 1)]
        if cfg.backend == "blas":
            self._init_blas(inst.blas_ops, inst.blas_plans)
        else:
            self._init_fft(inst.fft_ops, inst.halo_plans)
        self._bufs = {}
        self._canary_on = os.environ.get("KIFMM_CANARY", "0") == "1"
        self._canaries = []
        self._marks = None
        self.last_timings = {}
        self.last_m2l_calls = []

    # ------------------------------------------------------------ BLAS-M2L
    def _init_blas(self, ops, plans):
        import os
        self.blas = BlasDevice(ops, self.np_dtype, self.la)
        # M2L expansion folded with the down-solve's first factor: U^T U_dn
        self.blas.UTU = to_dev(np.asarray(ops.u, np.float64).T
                               @ np.asarray(self.inst.expansions.down_inv.u, np.float64),
                               self.np_dtype)
        self.blas_plan_dev = {l: upload_blas_plan(p) for l, p in plans.items()}
        # float32 engine path: TMA-fed sweep on dense sub-lattice arrays
        self.tma = self.blas.tc
        if self.tma:
            st, tt = self.inst.source_tree, self.inst.target_tree
            self.tma_plan = {l: tma_level_plan(st.level_keys(l), tt.level_keys(l), l)
                             for l in plans}

    def m2l_blas_level(self, lvl, mult, nrhs, check, solve=None, coarse_ctas=0,
                       projected=False, after_sweep=None):
        """Each level has its own scratch (qt, acc): levels run concurrently
        in the overlapped evaluate."""
        b = self._buffers(nrhs)
        qt, acc = b["qt_lv"][lvl], b["acc_lv"][lvl]
        if self.tma:
            plan = self.tma_plan[lvl]
            return self.blas.run_level_tma(plan, mult, self.n_src[lvl], self.n_tgt[lvl], nrhs,
                                           1.0 / self.side[lvl], qt, b["dense"][lvl], acc, solve,
                                           check=check, coarse_ctas=coarse_ctas,
                                           projected=projected,
                                           after_sweep=after_sweep)
        return self.blas.run_level(self.blas_plan_dev[lvl], mult, self.n_src[lvl],
                                   self.n_tgt[lvl], nrhs, 1.0 / self.side[lvl], check, qt, acc,
                                   solve=solve)

    # ------------------------------------------------------------- FFT-M2L
    def _init_fft(self, ops, plans):
        self.order = ops.order
        self.n_freq = ops.n_freq
        kh = np.ascontiguousarray(ops.khat)
        self.khat = to_dev(kh.view(np.float32 if kh.dtype == np.complex64 else np.float64))
        self.fft_plan_dev = {}
        for l, p in plans.items():
            sbox = np.full(p.n_src_clusters * 8, -1, dtype=np.int32)
            sbox[p.src_slot] = np.arange(p.src_slot.shape[0])
            tbox = np.full(p.n_tgt_clusters * 8, -1, dtype=np.int32)
            tbox[p.tgt_slot] = np.arange(p.tgt_slot.shape[0])
            self.fft_plan_dev[l] = dict(nsc=p.n_src_clusters, ntc=p.n_tgt_clusters,
                                        sbox=to_dev(sbox), tbox=to_dev(tbox),
                                        halo=to_dev(p.halo, np.int64),
                                        tiles=upload_hadamard_tiles(p.halo, p.src_color, p.tgt_color))

    def m2l_fft_level(self, lvl, mult, nrhs, check, plan=None):
        plan = plan if plan is not None else self.fft_plan_dev[lvl]
        b = self._buffers(nrhs)
        nsc, ntc = plan["nsc"], plan["ntc"]
        qh, ph = b["qhat_lv"][lvl], b["phat_lv"][lvl]
        qhat = qh[: 2 * self.n_freq * nsc * 8 * nrhs]
        phat = ph[: 2 * self.n_freq * ntc * 8 * nrhs]
        s = stream_handle()
        launch(f"kifmm_fft_forward_{self.sfx}", P(mult), nrhs, self.order, P(plan["sbox"]), nsc,
               None, 0, P(qhat), s)
        hadamard_tiled(self.sfx, self.khat, qhat, plan["tiles"], self.n_freq, nsc, ntc, nrhs,
                       phat, s)
        launch(f"kifmm_fft_inverse_{self.sfx}", P(phat), nrhs, self.order, P(plan["tbox"]), ntc,
                 1.0 / self.side[lvl], P(check), s)
        return 4

    # -------------------------------------------------------------- buffers
    # KIFMM_CANARY=1 (tests): every evaluate buffer gets CANARY guard
    # elements before and after it, filled with a sentinel; check_canaries()
    # reports any kernel write outside its buffer (compute-sanitizer is not
    # available on the B200 pool)
    CANARY = 4096

    def _alloc(self, n, dtype, zero=False):
        n = int(n)
        if not getattr(self, "_canary_on", False):
            return (torch.zeros if zero else torch.empty)(n, dtype=dtype, device=_dev())
        pad = self.CANARY
        full = torch.empty(n + 2 * pad, dtype=dtype, device=_dev())
        sentinel = -1.2345e30
        full.fill_(sentinel)
        inner = full[pad: pad + n]
        if zero:
            inner.zero_()
        self._canaries.append((full, n, sentinel))
        return inner

    def check_canaries(self):
        """[(buffer index, elements clobbered before, after)] for every guarded
        buffer whose guard elements changed (empty: no out-of-bounds write)."""
        torch.cuda.synchronize()
        bad = []
        for i, (full, n, sentinel) in enumerate(getattr(self, "_canaries", [])):
            pad = self.CANARY
            head = int((full[:pad] != sentinel).sum().item())
            tail = int((full[pad + n:] != sentinel).sum().item())
            if head or tail:
                bad.append((i, head, tail))
        return bad

    def _buffers(self, nrhs):
        if nrhs in self._bufs:
            return self._bufs[nrhs]
        T, dev = self.T, _dev()
        R = nrhs
        d = self.depth
        b = {}
        b["q"] = self._alloc(self.sx.shape[0] * R, T)
        b["src4"] = self._alloc(self.sx.shape[0] * R * 4, T)
        b["mult"] = [self._alloc(self.n_src[l] * R * self.n_e, T)
                     for l in range(d + 1)]
        b["loc"] = [self._alloc(self.n_tgt[l] * R * self.n_e, T)
                    for l in range(d + 1)]
        nmax_rows = max(max(self.n_src), max(self.n_tgt)) * R
        b["phi"] = self._alloc(max(nmax_rows * max(self.n_c, 1),
                                   max(self.n_tgt[:d] + [1]) * R * 8 * self.n_c), T)
        rmax = max(self.r_up, self.r_dn)
        b["tmp"] = self._alloc(max(nmax_rows, max(self.n_tgt[:d] + [1]) * 8 * R) * rmax, T)
        b["stack"] = self._alloc(max(self.n_src[2:d] + [1]) * R * 8 * self.n_e, T)
        # per-level M2L scratch (levels run concurrently in the overlapped
        # evaluate): check rows, and the BLAS (qt, acc) or FFT (qhat, phat) sets
        levels = list(range(2, d + 1))
        b["phi_lv"] = {l: self._alloc(max(self.n_tgt[l] * R * self.n_c, 1), T)
                       for l in levels}
        b["t_lv"] = {l: self._alloc(max(self.n_tgt[l] * R * self.r_fold, 1), T)
                     for l in levels}
        if self.cfg.backend == "blas":
            def acc_need(l):
                n = self.blas.acc_elems(self.n_tgt[l], R, self.blas_plan_dev[l]["n_tiles"])
                if self.tma:
                    n = max(n, self.blas.acc_elems(self.n_tgt[l], R, self.tma_plan[l]["n_tiles"],
                                                   tma=True, n_pairs=self.tma_plan[l]["n_pairs"]))
                return max(n, 1)
            qt_w = R * self.blas.kin * (3 if self.blas.tc else 1)
            b["qt_lv"] = {l: self._alloc(max(self.n_src[l], 1) * qt_w, T, zero=True)
                          for l in levels}
            b["acc_lv"] = {l: self._alloc(acc_need(l), T, zero=True) for l in levels}
            if self.tma:
                b["dense"] = {l: tuple(self._alloc(8 * R * p["h"] ** 3 * self.blas.kin, T,
                                                   zero=True) for _ in range(2))
                              for l, p in self.tma_plan.items()}
        else:
            fp = self.fft_plan_dev
            b["qhat_lv"] = {l: self._alloc(2 * self.n_freq * fp[l]["nsc"] * 8 * R, T)
                            for l in levels}
            b["phat_lv"] = {l: self._alloc(2 * self.n_freq * fp[l]["ntc"] * 8 * R, T)
                            for l in levels}
        b["out"] = self._alloc(self.tx.shape[0] * R, T)
        if self.mutual is not None:
            b["pmut"] = self._alloc(max(self.mutual["total"], 1) * R, T)
        b["qin"] = self._alloc(self.sx.shape[0] * R, torch.float64)
        self._bufs[nrhs] = b
        return b

    def _l2l_children_dense(self, lvl):
        """True when child c of parent p is target row 8p + c at level lvl for
        every parent (uniform trees), so the L2L output needs no row map."""
        if not hasattr(self, "_l2l_dense"):
            self._l2l_dense = {}
        if lvl not in self._l2l_dense:
            ch = np.asarray(self._tgt_child_np[lvl]).reshape(-1)
            self._l2l_dense[lvl] = bool(np.array_equal(ch, np.arange(ch.size)))
        return self._l2l_dense[lvl]

    def _l2l_rowmap(self, lvl, nrhs):
        """Row map of the L2L solve output (p, r, c) -> child row * R + r."""
        key = (lvl, nrhs)
        if key not in self._l2l_rowmaps:
            ch = self._tgt_child_np[lvl]                           # (n_par, 8)
            n_par = ch.shape[0]
            r = np.arange(nrhs)
            dest = ch[:, None, :] * nrhs + r[None, :, None]        # (n_par, R, 8)
            dest = np.where(ch[:, None, :] >= 0, dest, -1)
            self._l2l_rowmaps[key] = to_dev(dest.reshape(n_par * nrhs * 8), np.int32)
        return self._l2l_rowmaps[key]

    # ------------------------------------------------------------- evaluate
    def evaluate_device(self, q_dev, nrhs, timings=False, gradient=False):
        """Full evaluate from float64 charges on the device (caller order,
        (n_src, R) C-contiguous) to potentials on the device (caller order,
        (n_tgt, R), working dtype).  Returns the output tensor (a view of an
        internal buffer).

        With ``overlap`` the far-field pipeline runs on a high-priority stream
        and the near field on a low-priority one, so the block scheduler
        serves the (latency-bound) far-field kernels first and fills the
        rest of the machine with P2P work."""
        if self.overlap and not timings and _PROF is None:
            caller = torch.cuda.current_stream()
            self.hi_stream.wait_stream(caller)
            with torch.cuda.stream(self.hi_stream):
                res = self._evaluate(q_dev, nrhs, False, gradient, True)
            caller.wait_stream(self.hi_stream)
            return res
        return self._evaluate(q_dev, nrhs, timings, gradient, False)

    def _evaluate(self, q_dev, nrhs, timings, gradient, overlap):
        b = self._buffers(nrhs)
        R = nrhs
        s = stream_handle()
        d = self.depth
        n_e, n_c = self.n_e, self.n_c
        la, sfx = self.la, self.sfx
        ev = [] if timings else None
        # operator intervals recorded inside a captured graph (external
        # events: re-recorded by every replay; graph_timings reads them)
        marks = self._marks

        def mark(key):
            if marks is not None:
                e = torch.cuda.Event(enable_timing=True, external=True)
                e.record(torch.cuda.current_stream())
                marks.setdefault(key, []).append(e)

        def phase(name):
            set_tag(name)
            if ev is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ev.append((name, e))

        phase("p2m")
        mark("p2m")
        q = b["q"]
        launch(f"kifmm_gather_pack_{sfx}", P(q_dev), P(self.s_perm), P(self.sx), P(self.sy),
               P(self.sz), self.sx.shape[0], R, P(q), P(b["src4"]), s)
        # The near field (P2P) needs only the packed sources: with `overlap`
        # it runs on a low-priority side stream concurrently with the
        # far-field pipeline (mostly latency-bound small-level kernels), and
        # the L2P pass adds the far field at the end.  It is forked after the
        # upward pass: forked at once (after the pack or P2M), its CTAs fill
        # the machine and the P2M/M2M chain on the critical path waits for
        # free slots (config 2: 0.904 vs 0.892 ms).  Eager timing/profiling
        # passes run the near field in sequence.
        out = b["out"]
        nt = self.tx.shape[0]
        if gradient and "grad" not in b:
            b["grad"] = self._alloc(nt * R * 3, self.T)
        grad_ptr = [P(b["grad"])] if gradient else []
        leaf_name = f"kifmm_leaf_pass_grad_{sfx}" if gradient else f"kifmm_leaf_pass_{sfx}"

        guard_bit = 8 if self.p2p_guard else 0

        def leaf_args(parts):
            return [P(self.tx), P(self.ty), P(self.tz), P(self.t_start), P(self.t_count),
                    self.n_tgt[d], P(self.t_centers), P(self.equiv_base), n_e,
                    P(b["loc"][d]), P(b["src4"]), self.sx.shape[0], P(self.s_start),
                    P(self.s_count), P(self.near_off), P(self.near_leaf), R, P(self.t_perm),
                    parts | guard_bit, P(out)] + grad_ptr

        mut = self.mutual
        near_sorted = None
        if mut is not None and not gradient and sfx == "f32" and n_e <= 256:
            if "near_sorted" not in b:
                b["near_sorted"] = self._alloc(nt * R, self.T)
            near_sorted = b["near_sorted"]
        if mut is not None and gradient and "pmut4" not in b:
            b["pmut4"] = self._alloc(max(mut["total"], 1) * R * 4, self.T)

        def p2p_pass(stream):
            if mut is not None:
                # mutual near field into the partial-sum slots, then their
                # per-target totals into out (caller order)
                g_ = "grad_" if gradient else ""
                pm = b["pmut4"] if gradient else b["pmut"]
                launch(f"kifmm_p2p_mutual_{g_}{sfx}", P(self.tx), P(self.ty), P(self.tz),
                       self.n_tgt[d], P(b["src4"]), self.sx.shape[0], P(self.near_off),
                       P(mut["pack"]), P(mut["order"]), R, mut["total"], int(self.p2p_guard),
                       P(pm), stream)
                # float32 potential: totals in tree order (coalesced), added by
                # the final L2P pass, which alone un-permutes
                launch(f"kifmm_p2p_mutual_reduce_{g_}{sfx}", P(self.t_start), P(self.t_count),
                       self.n_tgt[d], R, None if near_sorted is not None else P(self.t_perm),
                       P(mut["base"]), P(mut["nlow"]), mut["total"], P(pm),
                       P(near_sorted) if near_sorted is not None else P(out), *grad_ptr, stream)
            else:
                launch(leaf_name, *leaf_args(2), stream)             # P2P, overwrite

        def l2p_final(stream):
            if near_sorted is not None:
                launch("kifmm_l2p_add_f32", P(self.tx), P(self.ty), P(self.tz), P(self.t_start),
                       P(self.t_count), self.n_tgt[d], P(self.t_centers), P(self.equiv_base), n_e,
                       P(b["loc"][d]), R, P(self.t_perm), P(near_sorted), P(out), stream)
            else:
                launch(leaf_name, *leaf_args(1 | 4), stream)         # L2P, accumulate

        side = self.side_stream

        def fork_p2p():
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                mark("p2p")
                p2p_pass(side.cuda_stream)
                mark("p2p")

        # P2M: check potentials, then the up_inv solve scaled by the leaf side.
        mult, phi, tmp = b["mult"], b["phi"], b["tmp"]
        nl = self.n_src[d]
        launch(f"kifmm_p2m_check_{sfx}", P(self.sx), P(self.sy), P(self.sz), P(q), R,
               P(self.s_start), P(self.s_count), nl, P(self.s_centers), P(self.check_base),
               n_c, P(phi), s)
        # float32, narrow operators (p <= 4), tensor-memory sweep: the solve and
        # the leaf level's M2L projection in one fused row chain (one launch
        # instead of three latency-bound GEMMs in front of the finest sweep)
        fused_p2m = (sfx == "f32" and self.cfg.backend == "blas" and self.tma
                     and self.blas.tmem and d >= 3 and max(n_c, n_e, self.blas.kin) <= 64)
        if fused_p2m:
            u, vals, vt = self.up_inv
            la.rowchain(nl * R, phi, n_c,
                        [(u, n_c, u.shape[1], vals, 1.0, None, 0, None, False),
                         (vt, u.shape[1], n_e, None, self.side[d], mult[d], n_e, None, False),
                         (self.blas.S, n_e, self.blas.kin, None, 1.0, b["dense"][d][0],
                          self.blas.kin, dense_rowmap(self.tma_plan[d], R), False)])
        else:
            la.chain(nl * R, phi, n_c, Linalg.solve_stages(self.up_inv, self.side[d]), mult[d],
                     n_e)
        mark("p2m")
        loc = b["loc"]
        calls = {}
        # Each level's M2L leaves its check potentials (x 1/side) in
        # phi_lv[l]; the L2L from the parent level adds its child check
        # potentials (x 0.5/side) into the same rows; one down_inv solve
        # (x side) then overwrites the locals.  The solve is linear, so this
        # equals the reference's two solves accumulated into the locals
        # (engine.py:355, 370) and saves one solve per level.
        rf = self.r_fold

        def m2l(lvl, after_sweep=None):
            # t_l = check_l . U_dn (rank rf) from the level's M2L
            n_t = self.n_tgt[lvl]
            t_l = b["t_lv"][lvl][: n_t * R * rf]
            if self.cfg.backend == "blas" and self.tma:
                calls[lvl] = self.m2l_blas_level(
                    lvl, mult[lvl], R, t_l,
                    coarse_ctas=self.coarse_ctas if overlap and lvl < d else 0,
                    projected=fused_p2m and lvl == d, after_sweep=after_sweep)
                return
            check = b["phi_lv"][lvl][: n_t * R * n_c]
            if self.cfg.backend == "blas":
                calls[lvl] = self.m2l_blas_level(lvl, mult[lvl], R, check)
            else:
                calls[lvl] = self.m2l_fft_level(lvl, mult[lvl], R, check)
            la.gemm(n_t * R, rf, n_c, 1.0, check, n_c, self.dn_u, rf, t_l, rf)

        def solve_level(lvl):
            # locals = t_l . diag(inv) V_dn^T x side (overwrite)
            n_t = self.n_tgt[lvl]
            t_l = b["t_lv"][lvl][: n_t * R * rf]
            la.gemm(n_t * R, n_e, rf, self.side[lvl], t_l, rf, self.dn_vv, n_e, loc[lvl], n_e)

        # With `overlap`, every level's M2L except the coarsest runs on its own
        # stream as soon as its multipoles exist (the finest level right after
        # P2M, level l after the M2M into l), concurrently with the M2M pass;
        # the main stream keeps only the dependent chain M2M -> M2L(2) ->
        # L2L(2->3) -> ... -> L2L(d-1->d), and each L2L into level l waits for
        # M2L(l) (both accumulate into loc[l]).  Every level has its own scratch.
        main = torch.cuda.current_stream()
        forked = {}

        def fork_m2l(lvl, after_sweep=None):
            st = self.level_streams[lvl]
            st.wait_stream(main)
            with torch.cuda.stream(st):
                mark("m2l")
                m2l(lvl, after_sweep)
                mark("m2l")
            forked[lvl] = st

        # the finest level's M2L is forked right after P2M (forking it after
        # the M2M pass, so the persistent sweep cannot hold the SMs the
        # latency-bound M2M chain needs, measured within +-1%)
        # The near field is released when the finest level's persistent sweep
        # ENDS.  Both are whole-GPU throughput kernels; a sweep CTA needs an
        # SM's whole shared memory, so near-field CTAs resident on an SM keep
        # the sweep off it (released together with the sweep - after its
        # projection - the sweep took 340 us instead of 282 and the evaluate
        # 850 us instead of 842; released after the upward pass, later still).
        # The M2M chain, the coarse levels and the L2L chain (small
        # latency-bound kernels on higher-priority streams) run in the near
        # field's shadow.  Measured bounds of this schedule at config 2: with
        # the coarse-level sweeps removed the evaluate takes 778 us, so their
        # ~40 us of tensor work costs 64 us; prefix (78) + finest sweep (282) +
        # near field (277) + L2P (52) = 689 us is the floor of the DAG.
        p2p_forked = False
        if overlap and d >= 3:
            if self.cfg.backend == "blas" and self.tma:
                fork_m2l(d, after_sweep=fork_p2p)
                p2p_forked = True
            else:
                fork_m2l(d)
        phase("m2m")
        mark("m2m")
        # M2M down to level 2 (levels 0-1 carry no M2L): children stacked in
        # the chain's loader, kernel product, then the up_inv solve.
        for lvl in range(d, 2, -1):
            n_par = self.n_src[lvl - 1]
            la.chain(n_par * R, mult[lvl], n_e,
                     [(self.m2mT, 8 * n_e, n_c, None, 1.0)]
                     + Linalg.solve_stages(self.up_inv, 1.0), mult[lvl - 1], n_e,
                     a_child=self.src_child[lvl], child_w=n_e, a_nrhs=R)
            if overlap and lvl - 1 >= 3:
                fork_m2l(lvl - 1)
        mark("m2m")
        if overlap and not p2p_forked:
            fork_p2p()
        for lvl in range(2, d + 1):
            n_t = self.n_tgt[lvl]
            phase(f"m2l{lvl}")
            if lvl not in forked and lvl not in calls:
                mark("m2l")
                m2l(lvl)
                mark("m2l")
            if lvl == 2:
                mark("m2l")
                solve_level(2)
                mark("m2l")
            if lvl < d:
                # the level's M2L check potentials must exist before the L2L
                # adds to them
                if lvl + 1 in forked:
                    main.wait_stream(forked[lvl + 1])
                else:
                    phase(f"m2l{lvl + 1}")
                    mark("m2l")
                    m2l(lvl + 1)
                    mark("m2l")
                phase(f"l2l{lvl}")
                mark("l2l")
                # child check potentials (parent row x 8 children x n_c) into
                # scratch, then added to the level's M2L check rows
                # child parts of t (parent row x 8 children x rf) into scratch,
                # then added to the level's M2L part
                t_c = b["t_lv"][lvl + 1][: self.n_tgt[lvl + 1] * R * rf]
                if R == 1 and self._l2l_children_dense(lvl + 1):
                    # every parent has its 8 children at rows 8p..8p+7: the
                    # GEMM accumulates straight into them (same roundings as
                    # the scratch + scatter-add below, one launch fewer)
                    la.gemm(n_t, 8 * rf, n_e, 0.5 / self.side[lvl + 1], loc[lvl], n_e,
                            self.l2lU, 8 * rf, t_c, 8 * rf, accumulate=True)
                else:
                    l2l_tmp = la.scratch(3, n_t * R * 8 * rf, self.T, t_c.device)
                    la.gemm(n_t * R, 8 * rf, n_e, 0.5 / self.side[lvl + 1], loc[lvl], n_e,
                            self.l2lU, 8 * rf, l2l_tmp, 8 * rf)
                    launch(f"kifmm_scatter_add_rows_{sfx}", P(l2l_tmp),
                           P(self._l2l_rowmap(lvl + 1, R)), n_t * R * 8, rf, P(t_c), s)
                solve_level(lvl + 1)
                mark("l2l")
        for st in forked.values():
            main.wait_stream(st)
        calls = [calls[l] for l in sorted(calls)]
        phase("leaf")
        if overlap:
            main.wait_stream(side)
            mark("l2p")
            l2p_final(s)
            mark("l2p")
        elif mut is not None:
            phase("p2p")
            mark("p2p")
            p2p_pass(s)
            mark("p2p")
            phase("l2p")
            mark("l2p")
            l2p_final(s)
            mark("l2p")
        else:
            mark("p2p")
            launch(leaf_name, *leaf_args(3), s)                      # fused L2P + P2P
            mark("p2p")
        phase("end")
        self.last_m2l_calls = calls
        self._events = ev
        if gradient:
            return out[: nt * R].view(nt, R), b["grad"][: nt * R * 3].view(nt, R, 3)
        return out[: nt * R].view(nt, R)

    # ------------------------------------------------------------ CUDA graph
    def graph_for(self, nrhs, gradient=False):
        """The whole evaluate captured once as a CUDA graph (one launch per
        evaluate instead of ~30 host-side kernel launches).  Returns
        (graph, static float64 charge buffer (n_src*R,), output tensor(s))."""
        if not hasattr(self, "_graphs"):
            self._graphs = {}
            self._graph_marks = {}
        key = (nrhs, bool(gradient))
        if key not in self._graphs:
            static_q = torch.zeros(self.sx.shape[0] * nrhs, dtype=torch.float64,
                                   device=self.sx.device)
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                for _ in range(2):                   # allocate buffers, cache plans
                    self.evaluate_device(static_q, nrhs, gradient=gradient)
            torch.cuda.current_stream().wait_stream(side)
            g = torch.cuda.CUDAGraph()
            # no garbage collection during the capture: a collected graph of
            # another instance would be destroyed mid-capture (not permitted,
            # invalidates this capture)
            import gc
            was_enabled = gc.isenabled()
            gc.disable()
            marks = {} if os.environ.get("KIFMM_GRAPH_TIMINGS", "1") != "0" else None
            self._marks = marks
            try:
                with torch.cuda.graph(g):
                    out = self.evaluate_device(static_q, nrhs, gradient=gradient)
            finally:
                self._marks = None
                if was_enabled:
                    gc.enable()
            self._graphs[key] = (g, static_q, out)
            self._graph_marks[key] = marks
        return self._graphs[key]

    def evaluate_graphed(self, q_dev, nrhs, gradient=False):
        """evaluate_device through the captured graph (q_dev: float64 device
        charges, caller order).  Returns the graph's output tensor(s)."""
        g, static_q, out = self.graph_for(nrhs, gradient)
        static_q.copy_(q_dev.reshape(-1))
        g.replay()
        return out

    def graph_timings(self, nrhs, gradient=False):
        """Operator seconds of the last replay of the (nrhs, gradient) graph,
        from the events recorded inside it, as a thunk (read on first use
        of ``FmmInstance.timings``; the replay must have completed).  The
        passes overlap on several streams, so the six intervals are each an
        operator's own span and may add up to more than the evaluate.  l2p
        is 0 when it is fused into the near-field pass."""
        marks = getattr(self, "_graph_marks", {}).get((nrhs, bool(gradient)))

        def read():
            t = {k: 0.0 for k in ("p2m", "m2m", "m2l", "l2l", "l2p", "p2p")}
            if not marks:
                return t
            for k, evs in marks.items():
                t[k] = sum(a.elapsed_time(b) for a, b in zip(evs[0::2], evs[1::2])) / 1e3
            return t
        return read

    # pageable host input: one (multi-threaded) torch host copy into a pinned
    # staging buffer, then an asynchronous H2D (measured on the B200 host,
    # 8 MB: 0.34 ms; a direct pageable copy 0.43 ms; a 4-thread chunked
    # numpy pipeline 0.9 ms)
    def _stage_pageable(self, src, dst):
        n = src.numel()
        stage = getattr(self, "_stage_buf", None)
        if stage is None or stage.numel() < n:
            stage = torch.empty(n, dtype=torch.float64, pin_memory=True)
            self._stage_buf = stage
        # the previous call's H2D from the staging buffer must be done
        ev = getattr(self, "_stage_done", None)
        if ev is not None:
            ev.synchronize()
        stage[:n].copy_(src)
        dst.copy_(stage[:n], non_blocking=True)
        self._stage_done = torch.cuda.Event()
        self._stage_done.record()

    def graph_timeline(self, nrhs, gradient=False):
        """[(operator, start ms, end ms)] of the last replay, relative to the
        start of its P2M (the graph's operator spans in time order)."""
        marks = getattr(self, "_graph_marks", {}).get((nrhs, bool(gradient))) or {}
        if "p2m" not in marks:
            return []
        t0 = marks["p2m"][0]
        out = [(k, t0.elapsed_time(a), t0.elapsed_time(b))
               for k, evs in marks.items() for a, b in zip(evs[0::2], evs[1::2])]
        return sorted(out, key=lambda x: x[1])

    def collect_timings(self):
        ev = getattr(self, "_events", None)
        if not ev:
            return {}
        ev[-1][1].synchronize()
        t = {k: 0.0 for k in ("p2m", "m2m", "m2l", "l2l", "l2p", "p2p")}
        for (n0, e0), (n1, e1) in zip(ev[:-1], ev[1:]):
            dt_s = e0.elapsed_time(e1) / 1e3
            key = "p2p" if n0 == "leaf" else ("m2l" if n0.startswith("m2l") else
                                               "l2l" if n0.startswith("l2l") else n0)
            t[key] += dt_s
        # without a separate l2p phase, L2P is fused into the leaf pass
        t["leaf_fused"] = 0.0 if any(n == "l2p" for n, _ in ev) else 1.0
        return t

    def evaluate_host(self, q_host: np.ndarray, timings=False, gradient=False):
        """Host charges (n_src, R) float64 in caller order -> host potentials.

        The charges are copied straight into the captured graph's input
        buffer, the graph is replayed, and the potentials are copied back
        (with ``timings=True`` the eager path runs instead, with per-phase
        CUDA events, to fill ``operator_timings``)."""
        R = q_host.shape[1]
        src = torch.from_numpy(np.ascontiguousarray(q_host, dtype=np.float64)).reshape(-1)
        if timings:
            b = self._buffers(R)
            qin = b["qin"][: q_host.size]
            qin.copy_(src)
            out = self.evaluate_device(qin, R, timings=True, gradient=gradient)
            self.last_timings = self.collect_timings()
            if gradient:
                return out[0].cpu().numpy().copy(), out[1].cpu().numpy().copy()
            return out.cpu().numpy().copy()
        g, static_q, out = self.graph_for(R, gradient)
        if src.is_pinned():
            # pinned host charges go over asynchronously, ordered before the replay
            static_q.copy_(src, non_blocking=True)
        else:
            self._stage_pageable(src, static_q)
        g.replay()
        outs = out if gradient else (out,)
        # results land in fresh pinned buffers (the caller owns the arrays; the
        # caching host allocator recycles a buffer only once it is released)
        host = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in outs]
        for h, o in zip(host, outs):
            h.copy_(o, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        res = tuple(h.numpy() for h in host)
        return res if gradient else res[0]


# ---------------------------------------------------------------- shims
def apply_level_host(ops, buckets, multipoles, n_targets, level_scale, counter=None):
    """Level-boundary drop-in for reference ``m2l_blas.apply_level``."""
    require_cuda()
    mult = np.ascontiguousarray(multipoles)
    dt = mult.dtype
    n_src, nrhs, n_e = mult.shape
    T = _NP2T[np.dtype(dt)]
    la = Linalg("f32" if dt == np.float32 else "f64")
    bd = BlasDevice(ops, dt, la)
    plan = upload_blas_plan(level_plan_from_buckets(buckets, n_targets))
    dev = _dev()
    m = to_dev(mult.reshape(n_src * nrhs, n_e))
    qt = torch.zeros(max(n_src, 1) * nrhs * bd.kin * 3, dtype=T, device=dev)
    acc = torch.zeros(max(bd.acc_elems(n_targets, nrhs, plan["n_tiles"]), 1), dtype=T, device=dev)
    check = torch.zeros(max(n_targets, 1) * nrhs * bd.n_c, dtype=T, device=dev)
    calls = bd.run_level(plan, m, n_src, n_targets, nrhs, level_scale, check, qt, acc)
    if counter is not None:
        counter.append(calls)
    return check[: n_targets * nrhs * bd.n_c].cpu().numpy().reshape(n_targets, nrhs, bd.n_c)


def upload_hadamard_tiles(halo_rows, src_color, tgt_color):
    """Device copy of plan_hadamard_tiles (the tiled Hadamard's plan)."""
    from .m2l_fft import plan_hadamard_tiles
    t = plan_hadamard_tiles(halo_rows, src_color, tgt_color)
    return dict(n_tiles=t.n_tiles, begin=to_dev(t.begin), src_off=to_dev(t.src_off),
                src=to_dev(t.src if t.src.size else np.zeros(1, np.int64)),
                slots=to_dev(t.slots if t.slots.size else np.zeros(1, np.int16)),
                tcol=to_dev(t.tcol if t.tcol.size else np.zeros(1, np.int16)))


def hadamard_tiled(sfx, khat, qhat, tiles, nf, nsc, ntc, nrhs, phat, stream, accumulate=0):
    """phat (=|+=) Hadamard M2L over a tile plan (csrc/hadamard.cu)."""
    cname = "c64" if sfx == "f32" else "c128"
    launch(f"kifmm_hadamard_tiled_{cname}", P(khat), P(qhat), P(tiles["begin"]),
           P(tiles["src_off"]), P(tiles["src"]), P(tiles["slots"]), P(tiles["tcol"]),
           tiles["n_tiles"], nf, nsc,
           ntc, nrhs, accumulate, P(phat), stream)


def m2l_fft_level_host(ops, plan, mult, level_scale):
    """Level-boundary drop-in for reference ``m2l_fft.m2l_fft_level``."""
    require_cuda()
    mult = np.ascontiguousarray(mult)
    dt = mult.dtype
    n_src, nrhs, n_e = mult.shape
    T = _NP2T[np.dtype(dt)]
    sfx = "f32" if dt == np.float32 else "f64"
    kh = np.ascontiguousarray(ops.khat.astype(np.complex64 if dt == np.float32 else np.complex128))
    khat = to_dev(kh.view(np.float32 if dt == np.float32 else np.float64))
    nsc, ntc = plan.n_src_clusters, plan.n_tgt_clusters
    sbox = np.full(nsc * 8, -1, dtype=np.int32)
    sbox[plan.src_slot] = np.arange(plan.src_slot.shape[0])
    tbox = np.full(ntc * 8, -1, dtype=np.int32)
    tbox[plan.tgt_slot] = np.arange(plan.tgt_slot.shape[0])
    n_tgt = plan.tgt_slot.shape[0]
    dev = _dev()
    nf = ops.n_freq
    qhat = torch.zeros(2 * nf * max(nsc, 1) * 8 * nrhs, dtype=T, device=dev)
    phat = torch.zeros(2 * nf * max(ntc, 1) * 8 * nrhs, dtype=T, device=dev)
    check = torch.zeros(max(n_tgt, 1) * nrhs * n_e, dtype=T, device=dev)
    s = stream_handle()
    m = to_dev(mult)
    keep = [to_dev(sbox), upload_hadamard_tiles(plan.halo, plan.src_color, plan.tgt_color),
            to_dev(tbox)]
    launch(f"kifmm_fft_forward_{sfx}", P(m), nrhs, ops.order, P(keep[0]), nsc, None, 0, P(qhat), s)
    hadamard_tiled(sfx, khat, qhat, keep[1], nf, nsc, ntc, nrhs, phat, s)
    launch(f"kifmm_fft_inverse_{sfx}", P(phat), nrhs, ops.order, P(keep[2]), ntc,
           float(level_scale), P(check), s)
    return check[: n_tgt * nrhs * n_e].cpu().numpy().reshape(n_tgt, nrhs, n_e)
