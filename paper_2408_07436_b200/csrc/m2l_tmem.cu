// BLAS-M2L sweep on tcgen05 with the A operand in tensor memory (float32,
// 3xTF32), persistent.
//
// Same contraction and numerics as m2l_tma.cu (3xTF32 products
// A_hi.B_hi + A_lo.B_hi + A_hi.B_lo, TMEM accumulator promoted into an IEEE
// fp32 accumulator every FLUSH_V vectors) over the same dense parity
// sub-lattice array of raw q~ rows, Q[p*R + r][ix][iy][iz][KP], and the same
// 4 x 4 x 8 same-parity target tiles (device.tma_level_plan).
//
// What changes is where A lives.  The TMA sweep stages every (tile, vector)
// source block in shared memory as TF32 hi and lo planes: 2 x 128 x KP x 4
// bytes written by TMA and read again by the MMA, which made it bound by
// shared-memory bandwidth (128 B/clk/SM) and by L2->SM bytes.  Here every
// loader thread owns one target row: it loads its source row for the vector
// straight into registers (ld.global.nc, L1-allocating: consecutive vectors
// of the locality-sorted order re-read 7/8 of the previous vector's rows),
// splits it into TF32 hi/lo in registers and stores both into TMEM with
// tcgen05.st (lane = row, column = K element).  The MMA reads A from TMEM;
// only the packed cores B = [B_hi | B_lo] (one bulk copy per vector) pass
// through shared memory.
//
// Per k-step (K = 8): D[:, 0:2KP] (+)= A_hi . [B_hi | B_lo]   (N = 2 KP)
//                     D[:, 0:N2]  +=  A_lo . B_hi             (N2 = KP rounded up to 16;
//   the columns KP..N2 of the second product land on A_lo . B_lo[0:N2-KP]
//   inside the B_lo half, which only adds the (tiny, correct) lo.lo term).
// The promotion sums D[:, c] + D[:, KP + c] into the IEEE accumulator.
//
// Persistent: gridDim.x CTAs (one per SM) walk the work items (rhs, tile,
// vector split) round-robin, keeping all pipelines running across items.
// Roles (448 threads): warp 0 lane 0 bulk-copies the cores (NS stages);
// warp 1 lane 0 issues tcgen05.mma.kind::tf32; warps 2..9 are two loader
// groups (group g serves the vectors with global index = g mod 2 into TMEM
// A buffer g); warps 10..13 promote and write the results.
#include <cuda.h>

#include <cstdlib>
#include <cstring>

#include "common.cuh"

using namespace kifmm;

namespace {

constexpr int TMT = 128;
constexpr int NG = 2;            // loader/MMA-issue groups, each with its own TMEM A and D
constexpr int NTHREADS = 64 + 128 * NG + 128;
constexpr int FLUSH_V = 4;
constexpr int BX = 4, BY = 4, BZ = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, bool sleep) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0, spins = 0;
  while (true) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) break;
    if (sleep) __nanosleep(64);
    if (++spins > (1u << 27)) __trap();    // watchdog: a lost arrive faults, never hangs
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint64_t desc_nosw(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// D[tmem] (+)= A[tmem] . B[smem]
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t addr, const uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
}
__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "r"(addr));
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                            int c2, int c3, int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"(smem_u32(bar))
      : "memory");
}
// bulk copy into the same offset of every CTA in cta_mask (and complete_tx on
// each one's barrier at the same offset)
__device__ __forceinline__ void bulk_copy_mc(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t b;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(x));
  return b;
}

struct TmemArgs {
  const float* q;                  // dense sub-lattice array (8*R, h, h, h, KP), raw fp32
  const float* bpair;              // (316, 2*KP*KP): [B_hi | B_lo] per vector, canonical layout
  int h, tx, ty, tz;
  const int32_t* tile_targets;     // (n_tiles*128)
  const int32_t* tile_ids;         // (n_tiles)
  const int32_t* pairs;            // (n_pairs, 2) tile slots of the same class per CTA pair
  const int32_t* class_tv;         // (8, 189) vector order per target class
  const int8_t* offsets;           // (316, 3)
  int n_tiles, n_pairs, nrhs, nsplit, jper, n_items, ns;
  int64_t ostride, ld;             // output: acc[(tgt*R + r)*ld + split*ostride + c]
  float* acc_out;
};

// Optional timeline of CTA 0 (tools/trace_tmem.py): clock64 per role and
// vector, set by kifmm_m2l_sweep_tmem_trace; null in normal runs.
__device__ long long* g_trace = nullptr;
__device__ int g_trace_h = 0;
constexpr int TRACE_N = 1024;
#define trace(ev, i)                                                                   \
  do {                                                                                 \
    if (trace_buf != nullptr && (i) < TRACE_N) trace_buf[(ev) * TRACE_N + (i)] = clock64(); \
  } while (0)

// Work item it -> (r, tile slot, split); its vector range [j0, j1).
struct Item {
  int slot, r, split, j0, nv;
};
// Items are (rhs, tile pair, split); CTA `rank` of the cluster takes tile
// pairs[pair][rank] (a class with an odd tile count repeats its last tile:
// both CTAs then compute and write the same rows).
__device__ __forceinline__ Item item_of(const TmemArgs& a, int it, int rank) {
  Item x;
  x.split = it % a.nsplit;
  const int rest = it / a.nsplit;
  const int pr = rest % a.n_pairs;
  x.slot = a.pairs[2 * pr + rank];
  x.r = rest / a.n_pairs;
  x.j0 = x.split * a.jper;
  x.nv = max(0, min(189, x.j0 + a.jper) - x.j0);
  return x;
}

// Each vector's source block arrives in shared memory by TMA (raw fp32,
// 128-byte swizzle, one 5-D box per 32 columns) together with its core pair
// [B_hi | B_lo] (bulk copy); each loader thread reads its row from there
// (conflict-free through the swizzle).
template <int KP>
__global__ void __launch_bounds__(NTHREADS, 1) m2l_sweep_tmem_kernel(
    const __grid_constant__ CUtensorMap tm, const TmemArgs a) {
  constexpr int N1 = 2 * KP;
  constexpr int N2 = (KP + 15) / 16 * 16;
  constexpr int NCH = (KP + 31) / 32;                                  // TMA boxes per vector
  constexpr uint32_t ABYTES = NCH * TMT * 128u;
  constexpr uint32_t BBYTES = 2u * KP * KP * 4u;
  constexpr uint32_t SBYTES = (ABYTES + BBYTES + 1023u) / 1024u * 1024u;
  // TMEM per group k: D_k (N1 columns) then A_k = [hi | lo] (2 KP columns)
  constexpr int GCOLS = N1 + 2 * KP;
  constexpr int NEED = NG * GCOLS;
  constexpr uint32_t TMEM_COLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128
                                 : NEED <= 256 ? 256 : 512;
  static_assert(NEED <= 512, "TMEM budget");
  static_assert(KP % 8 == 0 && N1 <= 256, "shape");

  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ns = a.ns;
  // clusters of 2 CTAs: both walk the same items (tile pairs of one class),
  // each loads its own source blocks and half of every core pair, which the
  // bulk copy multicasts into both CTAs' stages
  const int rank = (int)cluster_ctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();
  constexpr uint32_t BHALF = BBYTES / 2;
  long long* const trace_buf = (blockIdx.x == 0 && g_trace_h == a.h) ? g_trace : nullptr;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ns * SBYTES);
  uint64_t* empty = full + ns;
  uint64_t* done = empty + ns;          // [NG]: group k's MMAs of its last vector completed
  uint64_t* tfull = done + NG;          // [NG]: D_k holds a finished block
  uint64_t* tempty = tfull + NG;        // [NG]: D_k promoted
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NG);

  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);            // both CTAs' MMAs have read the stage
    }
    for (int k = 0; k < NG; ++k) {
      mbar_init(&done[k], 1);
      mbar_init(&tfull[k], 1);
      mbar_init(&tempty[k], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();                         // peer barriers initialised before any multicast
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int per_class = a.tx * a.ty * a.tz;

  if (warp == 0) {
    // ------------------------------------------- producer: A boxes + cores
    if (lane == 0) {
      int g = 0;
      for (int it = cid; it < a.n_items; it += ncl) {
        const Item x = item_of(a, it, rank);
        const int tile = a.tile_ids[x.slot];
        const int cls = tile / per_class;
        const int rem = tile - cls * per_class;
        const int ix0 = (rem / (a.ty * a.tz)) * BX, iy0 = ((rem / a.tz) % a.ty) * BY,
                  iz0 = (rem % a.tz) * BZ;
        const int px = (cls >> 2) & 1, py = (cls >> 1) & 1, pz = cls & 1;
        const int32_t* tv = a.class_tv + cls * 189 + x.j0;
        for (int v = 0; v < x.nv; ++v, ++g) {
          const int s = g % ns;
          if (g >= ns) mbar_wait(&empty[s], ((g / ns) - 1) & 1, false);
          trace(4, g);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                           smem_u32(&full[s])),
                       "r"(ABYTES + BBYTES)
                       : "memory");
          const int t = tv[v];
          unsigned char* sb = smem + s * SBYTES;
          const int ox = a.offsets[3 * t], oy = a.offsets[3 * t + 1], oz = a.offsets[3 * t + 2];
          const int qx = px + ox, qy = py + oy, qz = pz + oz;
          const int sp = ((qx & 1) << 2) | ((qy & 1) << 1) | (qz & 1);
          const int c4 = sp * a.nrhs + x.r;
#pragma unroll
          for (int c = 0; c < NCH; ++c)
            tma_load_5d(sb + c * TMT * 128, &tm, c * 32, iz0 + (qz >> 1), iy0 + (qy >> 1),
                        ix0 + (qx >> 1), c4, &full[s]);
          bulk_copy_mc(sb + ABYTES + rank * BHALF,
                       reinterpret_cast<const unsigned char*>(a.bpair + (int64_t)t * (2 * KP * KP)) +
                           rank * BHALF,
                       BHALF, &full[s], (uint16_t)0x3);
        }
      }
      // drain: the peer's MMA commits into this CTA's empty barriers arrive
      // asynchronously; wait for the last phase of every stage so no arrive
      // can land after this CTA has exited
      for (int gg = g - ns < 0 ? 0 : g - ns; gg < g; ++gg)
        mbar_wait(&empty[gg % ns], (gg / ns) & 1, true);
    }
    __syncwarp();
  } else if (warp >= 2 && warp < 2 + 4 * NG) {
    // ------------------------- loader + MMA-issue groups (vectors g = k mod NG)
    const int grp = (warp - 2) >> 2;
    const int q4 = warp & 3;                       // TMEM lane quarter of this warp
    const int m = q4 * 32 + lane;                  // tile row = TMEM lane
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    const bool issuer = (warp == 2 + 4 * grp) && lane == 0;
    const uint32_t dcol = tmem + (uint32_t)(grp * GCOLS);
    const uint32_t acol = dcol + N1;
    constexpr uint32_t idesc1 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N1 >> 3) << 17) |
                                ((uint32_t)(TMT >> 4) << 24);
    constexpr uint32_t idesc2 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N2 >> 3) << 17) |
                                ((uint32_t)(TMT >> 4) << 24);
    constexpr uint32_t SBO = (KP / 4) * 128;
    int nmine = 0;                                 // vectors this group has issued
    int blk = 0;                                   // blocks this group has committed
    int g = 0;
    for (int it = cid; it < a.n_items; it += ncl) {
      const Item x = item_of(a, it, rank);
      // this group's vectors of the item: v = v0, v0 + NG, ...
      const int v0 = ((grp - g) % NG + NG) % NG;
      int local = 0;                               // position inside the current block
      for (int v = v0; v < x.nv; v += NG) {
        const int gg = g + v;
        const int s = gg % ns;
        mbar_wait(&full[s], (gg / ns) & 1, false);
        if (m == 0) trace(0, gg);
        float4 cur[KP / 4];
        const unsigned char* sb = smem + s * SBYTES + m * 128;
#pragma unroll
        for (int i = 0; i < KP / 4; ++i)
          cur[i] = *reinterpret_cast<const float4*>(sb + (i >> 3) * (TMT * 128) +
                                                    (((i & 7) ^ (m & 7)) << 4));
        // previous MMAs of this group done: A_k (and, at a block start, D_k) reusable
        if (nmine > 0) mbar_wait(&done[grp], (nmine - 1) & 1, false);
        if (local == 0 && blk > 0) mbar_wait(&tempty[grp], (blk - 1) & 1, false);
        if (m == 0) trace(1, gg);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int c = 0; c < KP / 8; ++c) {
          uint32_t hv[8], lv[8];
          const float f[8] = {cur[2 * c].x,     cur[2 * c].y,     cur[2 * c].z,     cur[2 * c].w,
                              cur[2 * c + 1].x, cur[2 * c + 1].y, cur[2 * c + 1].z, cur[2 * c + 1].w};
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            // hi = TF32 round-to-nearest-away on the bit pattern; lo = x - hi is
            // exact in fp32 and enters the MMA truncated to TF32
            hv[i] = (__float_as_uint(f[i]) + 0x1000u) & 0xFFFFE000u;
            lv[i] = __float_as_uint(f[i] - __uint_as_float(hv[i]));
          }
          tmem_st8(acol + lane_base + c * 8, hv);
          tmem_st8(acol + lane_base + KP + c * 8, lv);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
        const bool last_of_block = (local == FLUSH_V - 1) || (v + NG >= x.nv);
        if (issuer) {
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          trace(3, gg);
          const uint32_t bb = smem_u32(smem + s * SBYTES + ABYTES);
#pragma unroll
          for (int ks = 0; ks < KP / 8; ++ks) {
            const uint64_t db = desc_nosw(bb + ks * 256, 128, SBO);
            mma_tf32_ts(dcol, acol + ks * 8, db, idesc1, local | ks);
            mma_tf32_ts(dcol, acol + KP + ks * 8, db, idesc2, 1);
          }
          mma_commit(&done[grp]);
          mma_commit_mc(&empty[s], (uint16_t)0x3);
          if (last_of_block) mma_commit(&tfull[grp]);
        }
        __syncwarp();
        ++nmine;
        if (last_of_block) {
          ++blk;
          local = 0;
        } else {
          ++local;
        }
        if (m == 0) trace(2, gg);
      }
      g += x.nv;
    }
  } else if (warp >= 2 + 4 * NG) {
    // --------------------------------- promotion of both groups' D, results
    const int q4 = warp & 3;
    const int m = q4 * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    float acc[KP];
    int cnt[NG];
#pragma unroll
    for (int k = 0; k < NG; ++k) cnt[k] = 0;
    int g = 0;
    for (int it = cid; it < a.n_items; it += ncl) {
      const Item x = item_of(a, it, rank);
#pragma unroll
      for (int c = 0; c < KP; ++c) acc[c] = 0.f;
      int nb[NG], nbmax = 0;
#pragma unroll
      for (int k = 0; k < NG; ++k) {
        const int v0 = ((k - g) % NG + NG) % NG;
        const int nk = x.nv > v0 ? (x.nv - v0 + NG - 1) / NG : 0;
        nb[k] = (nk + FLUSH_V - 1) / FLUSH_V;
        nbmax = max(nbmax, nb[k]);
      }
      for (int b = 0; b < nbmax; ++b) {
#pragma unroll
        for (int k = 0; k < NG; ++k) {
          if (b >= nb[k]) continue;
          mbar_wait(&tfull[k], cnt[k] & 1, true);
          if (m == 0 && k == 0) trace(5, cnt[0]);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t dcol = tmem + lane_base + (uint32_t)(k * GCOLS);
#pragma unroll
          for (int c = 0; c < KP / 8; ++c) {
            uint32_t u[8], w[8];
            tmem_ld8(dcol + c * 8, u);
            tmem_ld8(dcol + KP + c * 8, w);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 8; ++i)
              acc[c * 8 + i] += __uint_as_float(u[i]) + __uint_as_float(w[i]);
          }
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          mbar_arrive(&tempty[k]);
          if (m == 0 && k == 0) trace(6, cnt[0]);
          ++cnt[k];
        }
      }
      const int32_t tgt = a.tile_targets[(int64_t)x.slot * TMT + m];
      if (tgt >= 0) {
        float* o = a.acc_out + ((int64_t)tgt * a.nrhs + x.r) * a.ld + (int64_t)x.split * a.ostride;
#pragma unroll
        for (int c = 0; c < KP; c += 4)
          *reinterpret_cast<float4*>(o + c) = make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
      }
      g += x.nv;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();                         // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

// 5-D map over the dense sub-lattice array (k, iz, iy, ix, p*R + r); boxes of
// 32 k x (8, 4, 4) boxes x 1 plane, 128-byte swizzle, out-of-range -> zeros.
int make_map(CUtensorMap* tm, const float* base, int kp, int h, int64_t planes) {
  EncodeFn enc = encoder();
  if (!enc) return KIFMM_EARG;
  cuuint64_t dims[5] = {(cuuint64_t)kp, (cuuint64_t)h, (cuuint64_t)h, (cuuint64_t)h,
                        (cuuint64_t)planes};
  const cuuint64_t row = (cuuint64_t)kp * 4;
  cuuint64_t strides[4] = {row, row * h, row * h * h, row * h * h * h};
  cuuint32_t box[5] = {32, BZ, BY, BX, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult res = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS ? 0 : KIFMM_EARG;
}

template <int KP>
int launch_tmem(const TmemArgs& a0, cudaStream_t stream) {
  TmemArgs a = a0;
  static int ns_env = -1;
  if (ns_env < 0) {
    const char* e = getenv("KIFMM_TMEM_STAGES");
    ns_env = e ? atoi(e) : 4;
    if (ns_env < 2) ns_env = 2;
  }
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  int st = make_map(&tm, a.q, KP, a.h, 8 * (int64_t)a.nrhs);
  if (st) return st;
  const size_t sbytes = (((KP + 31) / 32) * TMT * 128 + 2ull * KP * KP * 4 + 1023) / 1024 * 1024;
  int ns = ns_env;
  while (ns > 2 && 1024 + ns * sbytes + 256 > 227 * 1024) --ns;
  a.ns = ns;
  const size_t smem = 1024 + ns * sbytes + (2 * ns + 3 * NG) * 8 + 16;
  const int ncl = a.n_items < sm_count() / 2 ? a.n_items : sm_count() / 2;
  set_max_smem((const void*)m2l_sweep_tmem_kernel<KP>, smem);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(2 * ncl, 1, 1);
  cfg.blockDim = dim3(NTHREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, m2l_sweep_tmem_kernel<KP>, tm, a);
  return e == cudaSuccess ? launch_status() : (int)e;
}

}  // namespace

extern "C" {

// Debug: record the timeline of CTA 0 of the following sweeps into buf
// (12 x 1024 int64 clock64 stamps; events documented at trace()); null stops.
int kifmm_m2l_sweep_tmem_trace(long long* buf, int64_t h) {
  cudaError_t e = cudaMemcpyToSymbol(g_trace, &buf, sizeof(buf));
  const int hh = (int)h;
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_trace_h, &hh, sizeof(hh));
  return e == cudaSuccess ? 0 : (int)e;
}

// Split of the 189-vector range (work items = R * n_pairs * nsplit) that
// balances the persistent CTA pairs: the smallest nsplit whose item count is
// within 4% of a whole number of waves (or the best found up to 16).
int kifmm_m2l_sweep_tmem_splits(int64_t n_pairs, int64_t nrhs, int64_t* nsplit) {
  if (n_pairs < 0 || nrhs < 1 || !nsplit) return KIFMM_EARG;
  const int g = sm_count() / 2;           // CTA pairs
  const int64_t n_tiles = n_pairs;
  int best = 1;
  double best_eff = 0;
  for (int s = 1; s <= 16; ++s) {
    const int jper = (189 + s - 1) / s;
    if ((s - 1) * jper >= 189) continue;           // would leave an empty piece
    const int nsp = s;
    const double items = (double)n_tiles * nrhs * nsp;
    const double waves = items / g;
    const double eff = waves / ((int64_t)(waves + 0.999999));
    // per-item fixed cost (first loads, result write) ~ 1/4 of a vector block
    const double cost = eff / (1.0 + 0.02 * nsp);
    if (cost > best_eff * 1.001) {
      best_eff = cost;
      best = s;
    }
  }
  *nsplit = best;
  return 0;
}

int kifmm_m2l_sweep_tmem_f32(const float* q, const float* bpair, int64_t kp, int64_t h,
                             const int32_t* tile_targets, const int32_t* tile_ids, int64_t n_tiles,
                             const int32_t* pairs, int64_t n_pairs, const int32_t* class_tv,
                             const int8_t* offsets, int64_t nrhs, int64_t nsplit, int64_t ostride,
                             float* acc, void* stream) {
  if (kp < 8 || kp % 8 || kp > 64 || n_tiles < 0 || nrhs < 1 || nsplit < 1 || nsplit > 189 ||
      h < 1 || ostride < kp || ostride % 4 || n_pairs < 0 || (n_tiles > 0 && n_pairs < 1))
    return KIFMM_EARG;
  if (n_tiles == 0) return 0;
  TmemArgs a;
  a.q = q;
  a.bpair = bpair;
  a.h = (int)h;
  a.tx = (int)((h + BX - 1) / BX);
  a.ty = (int)((h + BY - 1) / BY);
  a.tz = (int)((h + BZ - 1) / BZ);
  a.tile_targets = tile_targets;
  a.tile_ids = tile_ids;
  a.pairs = pairs;
  a.n_pairs = (int)n_pairs;
  a.class_tv = class_tv;
  a.offsets = offsets;
  a.n_tiles = (int)n_tiles;
  a.nrhs = (int)nrhs;
  a.nsplit = (int)nsplit;
  a.jper = (int)((189 + nsplit - 1) / nsplit);
  a.n_items = (int)(nrhs * n_pairs * nsplit);
  a.ostride = ostride;
  a.ld = nsplit * ostride;
  a.acc_out = acc;
  a.ns = 2;
  cudaStream_t s = (cudaStream_t)stream;
  switch (kp) {
    case 8: return launch_tmem<8>(a, s);
    case 16: return launch_tmem<16>(a, s);
    case 24: return launch_tmem<24>(a, s);
    case 32: return launch_tmem<32>(a, s);
    case 40: return launch_tmem<40>(a, s);
    case 48: return launch_tmem<48>(a, s);
    case 56: return launch_tmem<56>(a, s);
    case 64: return launch_tmem<64>(a, s);
  }
  return KIFMM_EARG;
}

}  // extern "C"
