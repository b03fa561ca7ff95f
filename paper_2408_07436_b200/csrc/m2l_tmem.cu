// BLAS-M2L sweep on tcgen05 with the A operand in tensor memory (float32,
// 3xTF32), persistent.
//
// Same contraction as m2l_tma.cu: per 4 x 4 x 8 same-parity target tile
// (device.tma_level_plan) and transfer vector t, the 128 source rows of the
// dense parity sub-lattice array of raw q~, Q[p*R + r][ix][iy][iz][KP], times
// the dense core D_t, in 3xTF32 (A_hi.B_hi + A_lo.B_hi + A_hi.B_lo) with the
// TMEM accumulator promoted into an IEEE fp32 accumulator every FLUSH_V
// vectors.
//
// What changes is where A lives.  The TMA sweep staged every (tile, vector)
// source block in shared memory as TF32 hi and lo planes (2 x 128 x KP x 4
// bytes written by TMA and read again by the MMA) plus the core pair, and
// was bound by shared-memory bandwidth.  Here the source block arrives raw by
// TMA (columns 0..31 in a 128-byte-swizzled box, the remaining KP - 32 in an
// exact-width box) and every loader thread reads its own row, splits it into
// TF32 hi/lo in registers and stores both into TMEM with tcgen05.st (lane =
// row, column = K element); the MMA reads A from TMEM, so only the core pair
// B = [B_hi | B_lo] is read from shared memory.
//
// Per k-step (K = 8): D[:, 0:2KP] (+)= A_hi . [B_hi | B_lo]   (N = 2 KP)
//                     D[:, 0:N2]  +=  A_lo . B_hi             (N2 = KP rounded up to 16;
//   the columns KP..N2 of the second product land on A_lo . B_lo[0:N2-KP]
//   inside the B_lo half, which only adds the (tiny, correct) lo.lo term).
// The promotion sums D[:, c] + D[:, KP + c] into the IEEE accumulator.
//
// Persistent: gridDim.x CTAs (one per SM) walk the work items (rhs, tile,
// vector split) round-robin through a ring of NS stages (source block + core
// pair, 53 KB at KP = 56).  Roles (352 threads): warp 0 lane 0 loads the
// stages; warps 1..4 and 5..8 are two loader groups taking alternate vectors:
// each loads, splits and stores its source rows into its own TMEM A buffer
// and hands the vector to its issuer warp (warps 9, 10: one thread issues the
// group's MMAs into the group's own TMEM accumulator), and promotes the
// accumulator into registers every FLUSH_V of its vectors; at the end of an
// item the two partial sums are combined through shared memory and group 0
// writes the result.  Groups never share a TMEM accumulator, so no MMA
// ordering between the issuing threads is needed - and the two groups'
// dependent MMA chains interleave on the tensor pipe, which hides the
// accumulate-to-accumulate latency of either (profiles/r2/sweep_bounds.md).
#include <cuda.h>

#include <cstdlib>
#include <cstring>

#include "common.cuh"

using namespace kifmm;

namespace {

constexpr int TMT = 128;
constexpr int NG = 2;             // groups per CTA (alternate vectors), each with its own TMEM A and D
constexpr int NTHREADS = 32 + 128 * NG + 32 * NG;   // producer, loader groups, issuer warps
#ifndef KIFMM_TMEM_FLUSH
#define KIFMM_TMEM_FLUSH 8
#endif
constexpr int FLUSH_V = KIFMM_TMEM_FLUSH;   // vectors between promotions of a TMEM accumulator
constexpr int BX = 4, BY = 4, BZ = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
#ifdef KIFMM_MBAR_DEBUG
__device__ unsigned g_mbar_dbg_n = 0;
__device__ unsigned g_mbar_dbg[256];
#endif
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
#ifdef KIFMM_MBAR_DEBUG
    if (++spins > (1u << 22)) {            // debug build: record the stuck wait and give up
      const unsigned i = atomicAdd(&g_mbar_dbg_n, 1u);
      if (i < 64) {
        g_mbar_dbg[4 * i] = blockIdx.x;
        g_mbar_dbg[4 * i + 1] = threadIdx.x;
        g_mbar_dbg[4 * i + 2] = a;
        g_mbar_dbg[4 * i + 3] = parity;
      }
      break;
    }
#else
    if (++spins > (1u << 27)) __trap();    // watchdog: a lost arrive faults, never hangs
#endif
  }
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

struct TmemArgs {
  const float* q;                  // dense sub-lattice array (8*R, h, h, h, KP), raw fp32
  const float* bpair;              // (316, 2*KP*KP): [B_hi | B_lo] per vector, canonical layout
  int h, tx, ty, tz;
  const int32_t* tile_targets;     // (n_tiles*128)
  const int32_t* tile_ids;         // (n_tiles)
  const int32_t* pairs;            // (n_pairs, 2) same-class tile slots handled by one CTA
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

// Work item it -> (r, tile slot, split): vectors [j0, j0 + nv) of the
// class list.
struct Item {
  int slot, r, split, j0, nv;
};
__device__ __forceinline__ Item item_of(const TmemArgs& a, int it) {
  Item x;
  x.split = it % a.nsplit;
  const int rest = it / a.nsplit;
  x.slot = rest % a.n_tiles;
  x.r = rest / a.n_tiles;
  x.j0 = x.split * a.jper;
  x.nv = max(0, min(189, x.j0 + a.jper) - x.j0);
  return x;
}

struct TileGeom {
  int cls, ix0, iy0, iz0, px, py, pz;
};
__device__ __forceinline__ TileGeom tile_geom(const TmemArgs& a, int slot) {
  const int per_class = a.tx * a.ty * a.tz;
  const int tile = a.tile_ids[slot];
  TileGeom t;
  t.cls = tile / per_class;
  const int rem = tile - t.cls * per_class;
  t.ix0 = (rem / (a.ty * a.tz)) * BX;
  t.iy0 = ((rem / a.tz) % a.ty) * BY;
  t.iz0 = (rem % a.tz) * BZ;
  t.px = (t.cls >> 2) & 1;
  t.py = (t.cls >> 1) & 1;
  t.pz = t.cls & 1;
  return t;
}

template <int KP>
__global__ void __launch_bounds__(NTHREADS, 1) m2l_sweep_tmem_kernel(
    const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm2,
    const TmemArgs a) {
  constexpr int N1 = 2 * KP;
  constexpr int N2 = (KP + 15) / 16 * 16;
  // source block: columns [0, 32) in a 128-byte-swizzled box, the rest
  // (KP - 32 columns) in a second box, swizzled when it is 32 wide and
  // linear (rows of (KP - 32) * 4 bytes, exact width) otherwise
  constexpr int W1 = KP > 32 ? KP - 32 : 0;
  constexpr bool SW1 = W1 == 32;
  constexpr uint32_t ABYTES = TMT * 128u + TMT * W1 * 4u;              // one source block
  constexpr uint32_t BBYTES = 2u * KP * KP * 4u;                       // one core pair
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
  long long* const trace_buf = (blockIdx.x == 0 && g_trace_h == a.h) ? g_trace : nullptr;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ns * SBYTES);
  uint64_t* empty = full + ns;          // the consuming group's MMAs have read the stage
  uint64_t* done = empty + ns;          // [NG]: group k's MMAs of its last vector completed
  uint64_t* aready = done + NG;         // [NG]: group k's 128 loaders have stored the vector's A
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aready + NG);   // + 16 B, then 4 KB reduction buffer

  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int k = 0; k < NG; ++k) {
      mbar_init(&done[k], 1);
      mbar_init(&aready[k], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
    if (W1) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm2)) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------ producer: source block + core pair
    if (lane == 0) {
      int g = 0;
      for (int it = blockIdx.x; it < a.n_items; it += gridDim.x) {
        const Item x = item_of(a, it);
        const TileGeom tg = tile_geom(a, x.slot);
        const int32_t* tv = a.class_tv + tg.cls * 189 + x.j0;
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
          const int qx = tg.px + ox, qy = tg.py + oy, qz = tg.pz + oz;
          const int sp = ((qx & 1) << 2) | ((qy & 1) << 1) | (qz & 1);
          const int cz = tg.iz0 + (qz >> 1), cy = tg.iy0 + (qy >> 1), cx = tg.ix0 + (qx >> 1);
          tma_load_5d(sb, &tm, 0, cz, cy, cx, sp * a.nrhs + x.r, &full[s]);
          if (W1) tma_load_5d(sb + TMT * 128, &tm2, 32, cz, cy, cx, sp * a.nrhs + x.r, &full[s]);
          bulk_copy(sb + ABYTES, a.bpair + (int64_t)t * (2 * KP * KP), BBYTES, &full[s]);
        }
      }
      // drain: the MMA commits on the stages arrive asynchronously; wait for
      // the last phase of every stage so none lands after this CTA exits
      for (int gg = g - ns < 0 ? 0 : g - ns; gg < g; ++gg)
        mbar_wait(&empty[gg % ns], (gg / ns) & 1, true);
    }
    __syncwarp();
  } else if (warp >= 1 && warp < 1 + 4 * NG) {
    // ------- group k: the vectors v = k (mod 2) of each item; load, issue,
    // promote into its own TMEM accumulator and registers, write its partial
    // result to split slot 2 * split + k
    const int grp = (warp - 1) >> 2;
    const int q4 = warp & 3;                       // TMEM lane quarter of this warp
    const int m = q4 * 32 + lane;                  // tile row = TMEM lane
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    const uint32_t dcol = tmem + (uint32_t)(grp * GCOLS);
    const uint32_t acol = dcol + N1;
    constexpr uint32_t idesc1 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N1 >> 3) << 17) |
                                ((uint32_t)(TMT >> 4) << 24);
    constexpr uint32_t idesc2 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N2 >> 3) << 17) |
                                ((uint32_t)(TMT >> 4) << 24);
    constexpr uint32_t SBO = (KP / 4) * 128;
    float acc[KP];
    int nmine = 0;                                 // vectors this group has issued
    int g = 0;
    for (int it = blockIdx.x; it < a.n_items; it += gridDim.x) {
      const Item x = item_of(a, it);
#pragma unroll
      for (int c = 0; c < KP; ++c) acc[c] = 0.f;
      int local = 0;                               // position in the group's current block
      for (int v = grp; v < x.nv; v += NG) {
        const int gg = g + v;
        const int s = gg % ns;
        mbar_wait(&full[s], (gg / ns) & 1, false);
        if (m == 0) trace(grp == 0 ? 0 : 5, gg);
        // this thread's source row -> TF32 hi (round-to-nearest-away on the bit
        // pattern) and lo = x - hi (exact in fp32; enters the MMA truncated to
        // TF32), in registers before waiting for the TMEM buffers
        uint32_t hv[KP], lv[KP];
        const unsigned char* sb = smem + s * SBYTES;
        auto split4 = [&](int i, const float4& c4) {
          const float f[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            hv[4 * i + j] = (__float_as_uint(f[j]) + 0x1000u) & 0xFFFFE000u;
            lv[4 * i + j] = __float_as_uint(f[j] - __uint_as_float(hv[4 * i + j]));
          }
        };
#pragma unroll
        for (int i = 0; i < (KP < 32 ? KP / 4 : 8); ++i)
          split4(i, *reinterpret_cast<const float4*>(sb + m * 128 + (((i & 7) ^ (m & 7)) << 4)));
        if (SW1) {
#pragma unroll
          for (int i = 8; i < KP / 4; ++i)
            split4(i, *reinterpret_cast<const float4*>(sb + TMT * 128 + m * 128 +
                                                       (((i & 7) ^ (m & 7)) << 4)));
        } else {
          // linear second box: rows W1 * 4 bytes apart (measured faster than
          // a conflict-free split into 16- and 8-column boxes with the 64- and
          // 32-byte swizzles: 259 vs 265 us, one TMA fewer per stage; and
          // than swapped chunk pairs: 284 vs 303 us)
#pragma unroll
          for (int i = 8; i < KP / 4; ++i)
            split4(i, *reinterpret_cast<const float4*>(sb + TMT * 128 + m * (W1 * 4) + (i - 8) * 16));
        }
        if (m == 0 && grp == 0) trace(2, gg);
        // this group's previous MMAs done: A_k reusable (and D_k promoted below)
        if (nmine > 0) mbar_wait(&done[grp], (nmine - 1) & 1, false);
        if (m == 0) trace(grp == 0 ? 1 : 6, gg);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int c = 0; c < KP / 8; ++c) {
          tmem_st8(acol + lane_base + c * 8, *reinterpret_cast<const uint32_t(*)[8]>(&hv[c * 8]));
          tmem_st8(acol + lane_base + KP + c * 8, *reinterpret_cast<const uint32_t(*)[8]>(&lv[c * 8]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        if (m == 0 && grp == 0) trace(7, gg);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        // hand the vector over to the group's issuer warp and go on to the
        // next source block (the issuing thread waits on the tensor pipe for
        // ~1100 clk per vector: as a loader thread it held its warp - and
        // through a group barrier the whole group - back)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&aready[grp]))
                     : "memory");
        __syncwarp();
        ++nmine;
        const bool last_of_block = local == FLUSH_V - 1 || v + NG >= x.nv;
        local = last_of_block ? 0 : local + 1;
        if (last_of_block) {
          // promote D_k: wait for this block's last MMAs, add into registers;
          // the next vector's MMA overwrites D_k only after the group barrier
          if (m == 0 && grp == 0) trace(8, gg);
          mbar_wait(&done[grp], (nmine - 1) & 1, false);
          if (m == 0 && grp == 0) trace(10, gg);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
          for (int c = 0; c < KP / 8; ++c) {
            uint32_t u[8], w[8];
            tmem_ld8(dcol + lane_base + c * 8, u);
            tmem_ld8(dcol + lane_base + KP + c * 8, w);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 8; ++i)
              acc[c * 8 + i] += __uint_as_float(u[i]) + __uint_as_float(w[i]);
          }
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          if (m == 0 && grp == 0) trace(11, gg);
        }
      }
      // combine the groups' partial sums in shared memory, 8 columns at a
      // time, and let group 0 write the item's result (one output slot per
      // vector split)
      float4* red = reinterpret_cast<float4*>(tmem_slot + 4);     // 128 x 8 floats
#pragma unroll
      for (int c = 0; c < KP; c += 8) {
#pragma unroll
        for (int g2 = 1; g2 < NG; ++g2) {
          if (grp == g2) {
            red[2 * m] = make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
            red[2 * m + 1] = make_float4(acc[c + 4], acc[c + 5], acc[c + 6], acc[c + 7]);
          }
          asm volatile("bar.sync %0, %1;" ::"r"(1 + NG), "r"(128 * NG) : "memory");
          if (grp == 0) {
            const float4 u = red[2 * m], w = red[2 * m + 1];
            acc[c] += u.x;
            acc[c + 1] += u.y;
            acc[c + 2] += u.z;
            acc[c + 3] += u.w;
            acc[c + 4] += w.x;
            acc[c + 5] += w.y;
            acc[c + 6] += w.z;
            acc[c + 7] += w.w;
          }
          asm volatile("bar.sync %0, %1;" ::"r"(1 + NG), "r"(128 * NG) : "memory");
        }
      }
      const int32_t tgt = a.tile_targets[(int64_t)x.slot * TMT + m];
      if (grp == 0 && tgt >= 0) {
        float* o = a.acc_out + ((int64_t)tgt * a.nrhs + x.r) * a.ld + (int64_t)x.split * a.ostride;
#pragma unroll
        for (int c = 0; c < KP; c += 4)
          *reinterpret_cast<float4*>(o + c) = make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
      }
      g += x.nv;
    }
  }
  else if (warp >= 1 + 4 * NG) {
    // ------- issuer warp of group k: per vector of the group, wait for the
    // loaders' A, issue the MMAs into D_k, commit (A_k / D_k free, stage free)
    const int grp = warp - (1 + 4 * NG);
    if (lane == 0) {
      const uint32_t dcol = tmem + (uint32_t)(grp * GCOLS);
      const uint32_t acol = dcol + N1;
      constexpr uint32_t idesc1 = (1u << 4) | (2u << 7) | (2u << 10) |
                                  ((uint32_t)(N1 >> 3) << 17) | ((uint32_t)(TMT >> 4) << 24);
      constexpr uint32_t idesc2 = (1u << 4) | (2u << 7) | (2u << 10) |
                                  ((uint32_t)(N2 >> 3) << 17) | ((uint32_t)(TMT >> 4) << 24);
      constexpr uint32_t SBO = (KP / 4) * 128;
      int g = 0, nmine = 0;
      for (int it = blockIdx.x; it < a.n_items; it += gridDim.x) {
        const Item x = item_of(a, it);
        int local = 0;
        for (int v = grp; v < x.nv; v += NG) {
          const int gg = g + v;
          const int s = gg % ns;
          mbar_wait(&full[s], (gg / ns) & 1, false);        // the stage's core pair has landed
          mbar_wait(&aready[grp], nmine & 1, false);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (grp == 0) trace(3, gg);
          const uint32_t bb = smem_u32(smem + s * SBYTES + ABYTES);
#pragma unroll
          for (int ks = 0; ks < KP / 8; ++ks) {
            const uint64_t db = desc_nosw(bb + ks * 256, 128, SBO);
            mma_tf32_ts(dcol, acol + ks * 8, db, idesc1, local | ks);
            mma_tf32_ts(dcol, acol + KP + ks * 8, db, idesc2, 1);
          }
          mma_commit(&done[grp]);
          mma_commit(&empty[s]);
          if (grp == 0) trace(9, gg);
          ++nmine;
          const bool last_of_block = local == FLUSH_V - 1 || v + NG >= x.nv;
          local = last_of_block ? 0 : local + 1;
        }
        g += x.nv;
      }
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

int sm_count() { return device_sm_count(); }

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
// `width` k x (8, 4, 4) boxes x 1 plane with the given swizzle (the row of the
// box, width * 4 bytes, equals the swizzle span), out-of-range -> zeros.
int make_map(CUtensorMap* tm, const float* base, int kp, int h, int64_t planes, int width,
             CUtensorMapSwizzle swizzle) {
  EncodeFn enc = encoder();
  if (!enc) return KIFMM_EARG;
  cuuint64_t dims[5] = {(cuuint64_t)kp, (cuuint64_t)h, (cuuint64_t)h, (cuuint64_t)h,
                        (cuuint64_t)planes};
  const cuuint64_t row = (cuuint64_t)kp * 4;
  cuuint64_t strides[4] = {row, row * h, row * h * h, row * h * h * h};
  cuuint32_t box[5] = {(cuuint32_t)width, BZ, BY, BX, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult res = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swizzle,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS ? 0 : KIFMM_EARG;
}

template <int KP>
int launch_tmem(const TmemArgs& a0, cudaStream_t stream) {
  TmemArgs a = a0;
  constexpr int W1 = KP > 32 ? KP - 32 : 0;
  CUtensorMap tm, tm2;
  memset(&tm, 0, sizeof(tm));
  memset(&tm2, 0, sizeof(tm2));
  const int64_t planes = 8 * (int64_t)a.nrhs;
  int st = make_map(&tm, a.q, KP, a.h, planes, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!st && W1 == 32) st = make_map(&tm2, a.q, KP, a.h, planes, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!st && W1 && W1 != 32)
    st = make_map(&tm2, a.q, KP, a.h, planes, W1, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st) return st;
  constexpr int ns_env = 4;             // config 2 on B200: 4 stages 259 us, 3: 279 us, 2: 351 us
  const size_t sbytes = ((size_t)TMT * 128 + (size_t)TMT * W1 * 4 + 2ull * KP * KP * 4 + 1023) /
                        1024 * 1024;
  int ns = ns_env;
  while (ns > 2 && 1024 + ns * sbytes + 256 + 4096 > 227 * 1024) --ns;
  // an even ring: stage s is then always consumed by the same group (vector
  // g -> stage g % ns, group g % 2).  With an odd ring the two groups
  // alternate on every stage, and repeated fresh evaluates at ns = 3 gave
  // wrong sums on a few tile-vectors (4 of 40) and occasional launch faults;
  // ns = 2 and ns = 4 gave none in 180 (tools/stress_overlap.py).
  if (ns & 1) --ns;
  a.ns = ns;
  const size_t smem = 1024 + ns * sbytes + (2 * ns + 2 * NG) * 8 + 16 + 4096;
  // persistent CTAs: one per SM (capping the grid to leave SMs to the
  // other streams' kernels measured within +-1%)
  const int g_max = sm_count();
  const int grid = a.n_items < g_max ? a.n_items : g_max;
  set_max_smem((const void*)m2l_sweep_tmem_kernel<KP>, smem);
  m2l_sweep_tmem_kernel<KP><<<grid, NTHREADS, smem, stream>>>(tm, tm2, a);
  return launch_status();
}

}  // namespace

extern "C" {

#ifdef KIFMM_MBAR_DEBUG
int kifmm_mbar_debug_read(unsigned* host) {
  cudaMemcpyFromSymbol(host, g_mbar_dbg_n, sizeof(unsigned));
  return (int)cudaMemcpyFromSymbol(host + 1, g_mbar_dbg, sizeof(g_mbar_dbg));
}
#endif

// Debug: record the timeline of CTA 0 of the following sweeps into buf
// (12 x 1024 int64 clock64 stamps; events documented at trace()); null stops.
int kifmm_m2l_sweep_tmem_trace(long long* buf, int64_t h) {
  cudaError_t e = cudaMemcpyToSymbol(g_trace, &buf, sizeof(buf));
  const int hh = (int)h;
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_trace_h, &hh, sizeof(hh));
  return e == cudaSuccess ? 0 : (int)e;
}

// Split of the 189-vector range (work items = R * n_tiles * nsplit) that
// balances the persistent CTAs: the best whole-wave fill, discounted by the
// per-item fixed cost (pipeline fill, result write).
int kifmm_m2l_sweep_tmem_splits(int64_t n_tiles, int64_t n_pairs, int64_t nrhs,
                                int64_t* nsplit) {
  if (n_tiles < 0 || n_pairs < 0 || nrhs < 1 || !nsplit) return KIFMM_EARG;
  const int g = sm_count();
  int best = 1;
  double best_eff = 0;
  for (int s = 1; s <= 16; ++s) {
    const int jper = (189 + s - 1) / s;
    if ((s - 1) * jper >= 189) continue;           // would leave an empty piece
    const double items = (double)n_tiles * nrhs * s;
    const double waves = items / g;
    const double eff = waves / ((int64_t)(waves + 0.999999));
    const double cost = eff / (1.0 + 0.02 * s);
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
  a.nrhs = (int)nrhs;
  a.nsplit = (int)nsplit;
  a.jper = (int)((189 + nsplit - 1) / nsplit);
  a.n_tiles = (int)n_tiles;
  a.n_items = (int)(nrhs * n_tiles * nsplit);
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
