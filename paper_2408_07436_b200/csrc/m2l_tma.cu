// BLAS-M2L sweep on tcgen05 fed by TMA box loads (float32, 3xTF32).
//
// Same contraction and numerics as m2l_tc.cu (3xTF32 products, TMEM
// accumulator promoted into an IEEE fp32 accumulator every FLUSH_V vectors,
// 189 vectors in ascending canonical order per parity class, split pieces
// summed by the caller), but the source rows are no longer gathered.
//
// Layout.  The projected multipoles q~ of a level (grid n = 2^l, h = n/2)
// are kept in a dense parity sub-lattice array
//     Q[p*R + r][ix][iy][iz][k],   box anchor = (2 ix + px, 2 iy + py, 2 iz + pz)
// (zero rows for pruned boxes).  A tile is a 4 x 4 x 8 block of same-parity
// (class p) targets, i in [i0, i0 + (4,4,8)).  The source of target 2i + p
// through vector t is 2i + p + t, i.e. sub-lattice p' = (p + t) & 1 at
// i' = i + ((p + t) >> 1): for every vector the tile's 128 sources are ONE
// 4 x 4 x 8 box of Q[p'], fetched by a single 5-D TMA load (128B swizzle,
// out-of-range boxes zero-filled by the TMA unit = absent sources).
//
// Roles (192 threads): warp 0 lane 0 issues the TMA loads (A_hi, A_lo) and
// the bulk copies of the core blocks (B_hi, B_lo) per stage; warp 1 lane 0
// issues tcgen05.mma.kind::tf32; warps 2..5 promote the TMEM accumulator and
// write the result.
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"

using namespace kifmm;

namespace {

constexpr int TMT = 128;        // targets per tile = MMA M
constexpr int KC = 32;          // K (floats) per stage = one 128-byte swizzle row
constexpr int NTHREADS = 192;
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
    if (sleep) __nanosleep(128);
    if (++spins > (1u << 26)) __trap();    // watchdog: a lost arrive faults, never hangs
  }
}
__device__ __forceinline__ uint64_t desc_nosw(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// K-major, 128-byte swizzle: 8-row x 128-byte atoms, SBO = 1024 between atoms.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;                        // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;              // SBO
  d |= (uint64_t)1 << 46;                        // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                        // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}
__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
        "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]),
        "r"(v[14]), "r"(v[15]));
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
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct TmaArgs {
  const float* bhi;
  const float* blo;
  int kin, n_out, stages, h;
  int tx, ty, tz;                  // tiles per class along x, y, z
  const int32_t* tile_targets;     // (n_tiles*128) target row or -1
  const int32_t* tile_ids;         // (n_tiles) linear tile id (class-major) of each launched tile
  const int32_t* class_tv;         // (8, 189)
  const int8_t* offsets;           // (316, 3)
  int64_t nrhs;
  int nsplit, jper;
  int split_smem;                  // 1: A arrives raw (fp32), hi/lo formed in shared memory
  int mma2;                        // 1: two MMAs per k-step, A_hi x [B_hi | B_lo] (N = 2 n_out)
  int nbuf;                        // TMEM accumulator buffers (2: MMA overlaps the promotion)
  float* acc_out;
};

__global__ void __launch_bounds__(NTHREADS, 1) m2l_sweep_tma_kernel(
    const __grid_constant__ CUtensorMap tm_hi, const __grid_constant__ CUtensorMap tm_lo,
    const TmaArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  // 1024-byte alignment for the swizzled A tiles
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kin = a.kin, n_out = a.n_out, stages = a.stages;
  const int nchunks = (kin + KC - 1) / KC;
  const uint32_t a_bytes = TMT * KC * 4;                 // 16 KB
  const uint32_t b_bytes = (uint32_t)n_out * KC * 4;
  const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* ready = empty + stages;                      // A hi/lo formed (split_smem)
  uint64_t* tfull = ready + stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int64_t slot = blockIdx.x;                       // launched tile
  const int tile = a.tile_ids[slot];
  const int per_class = a.tx * a.ty * a.tz;
  const int cls = tile / per_class;
  const int rem = tile - cls * per_class;
  const int ix0 = (rem / (a.ty * a.tz)) * BX, iy0 = ((rem / a.tz) % a.ty) * BY,
            iz0 = (rem % a.tz) * BZ;
  const int px = (cls >> 2) & 1, py = (cls >> 1) & 1, pz = cls & 1;
  const int64_t r = blockIdx.y;
  const int split = blockIdx.z;
  const int j0 = split * a.jper, j1 = min(189, j0 + a.jper);
  const int nvec = max(0, j1 - j0);
  const int nsteps = nvec * nchunks;
  const int nblocks = (nvec + FLUSH_V - 1) / FLUSH_V;
  const int32_t* tv_list = a.class_tv + cls * 189;
  // accumulator buffers of width dw (n_out, or 2 n_out in the 2-MMA form:
  // [A_hi B_hi + A_lo B_hi | A_hi B_lo]) x 2 + the IEEE accumulator
  const int dw = a.mma2 ? 2 * n_out : n_out;
  const int nbuf = a.nbuf;
  const uint32_t need = (uint32_t)(nbuf * dw) + (uint32_t)n_out;
  const uint32_t tmem_cols = need <= 64 ? 64 : need <= 128 ? 128 : need <= 256 ? 256 : 512;

  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&ready[s], 128);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tfull[1], 1);
    mbar_init(&tempty[0], 128);
    mbar_init(&tempty[1], 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_hi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_lo)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      for (int st = 0; st < nsteps; ++st) {
        const int stage = st % stages;
        const int round = st / stages;
        if (round > 0) mbar_wait(&empty[stage], (round - 1) & 1, false);
        const int j = j0 + st / nchunks, c = st % nchunks;
        const int kc = min(KC, kin - c * KC);
        const int t = tv_list[j];
        const int ox = a.offsets[3 * t], oy = a.offsets[3 * t + 1], oz = a.offsets[3 * t + 2];
        const int qx = px + ox, qy = py + oy, qz = pz + oz;    // source anchor offsets
        const int sp = ((qx & 1) << 2) | ((qy & 1) << 1) | (qz & 1);
        const int sx = ix0 + (qx >> 1), sy = iy0 + (qy >> 1), sz = iz0 + (qz >> 1);
        unsigned char* sb = smem + stage * stage_bytes;
        const uint32_t bb = (uint32_t)(n_out * kc * 4);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         smem_u32(&full[stage])),
                     "r"((a.split_smem ? 1 : 2) * a_bytes + 2 * bb)
                     : "memory");
        const int c4 = sp * (int)a.nrhs + (int)r;
        tma_load_5d(sb, &tm_hi, c * KC, sz, sy, sx, c4, &full[stage]);
        if (!a.split_smem) tma_load_5d(sb + a_bytes, &tm_lo, c * KC, sz, sy, sx, c4, &full[stage]);
        const int64_t boff = (int64_t)t * n_out * kin + (int64_t)n_out * KC * c;
        bulk_copy(sb + 2 * a_bytes, a.bhi + boff, bb, &full[stage]);
        bulk_copy(sb + 2 * a_bytes + bb, a.blo + boff, bb, &full[stage]);   // B_lo follows B_hi
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ----------------------------------------------------------- MMA issue
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n_out >> 3) << 17) |
                           ((uint32_t)(TMT >> 4) << 24);
    const uint32_t idesc2 = (1u << 4) | (2u << 7) | (2u << 10) |
                            ((uint32_t)((2 * n_out) >> 3) << 17) | ((uint32_t)(TMT >> 4) << 24);
    if (lane == 0) {
      int st = 0;
      for (int bi = 0; bi < nblocks; ++bi) {
        const int buf = bi % nbuf;
        if (bi >= nbuf) mbar_wait(&tempty[buf], ((bi / nbuf) - 1) & 1, false);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dcol = tmem + (uint32_t)(buf * dw);
        const int vend = min(nvec, (bi + 1) * FLUSH_V);
        uint32_t acc_flag = 0;
        for (; st < vend * nchunks; ++st) {
          const int stage = st % stages;
          mbar_wait(a.split_smem ? &ready[stage] : &full[stage], (st / stages) & 1, false);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const int c = st % nchunks;
          const int kc = min(KC, kin - c * KC);
          const uint32_t base = smem_u32(smem + stage * stage_bytes);
          const uint32_t a_hi = base, a_lo = base + a_bytes;
          const uint32_t b_hi = base + 2 * a_bytes;
          const uint32_t b_lo = b_hi + (uint32_t)(n_out * kc * 4);   // n-groups continue into B_lo
          const uint32_t sbo_b = (uint32_t)(kc / 4) * 128;
          for (int ks = 0; ks < kc / 8; ++ks) {
            const uint32_t ka = ks * 32;          // K offset inside the 128-byte swizzle row
            const uint32_t kb = ks * 256;         // two 128-byte core matrices along K
            if (a.mma2) {
              // [D | D'] = A_hi . [B_hi | B_lo] (one read of A_hi), then D += A_lo . B_hi
              mma_tf32(dcol, desc_sw128(a_hi + ka), desc_nosw(b_hi + kb, 128, sbo_b), idesc2,
                       acc_flag);
              acc_flag = 1;
              mma_tf32(dcol, desc_sw128(a_lo + ka), desc_nosw(b_hi + kb, 128, sbo_b), idesc, 1);
            } else {
              mma_tf32(dcol, desc_sw128(a_lo + ka), desc_nosw(b_hi + kb, 128, sbo_b), idesc,
                       acc_flag);
              acc_flag = 1;
              mma_tf32(dcol, desc_sw128(a_hi + ka), desc_nosw(b_lo + kb, 128, sbo_b), idesc, 1);
              mma_tf32(dcol, desc_sw128(a_hi + ka), desc_nosw(b_hi + kb, 128, sbo_b), idesc, 1);
            }
          }
          mma_commit(&empty[stage]);
        }
        mma_commit(&tfull[buf]);
      }
    }
    __syncwarp();
  } else {
    // ------------------- accumulator warps (2..5): A hi/lo split, promotion
    const int sub = warp & 3;
    const int m = sub * 32 + lane;
    const uint32_t lane_base = (uint32_t)(sub * 32) << 16;
    const uint32_t acc_col = tmem + lane_base + (uint32_t)(nbuf * dw);
    const int ct = tid - 64;                               // 0..127 converter thread
    auto promote = [&](int bi) {
      const int buf = bi % nbuf;
      mbar_wait(&tfull[buf], (bi / nbuf) & 1, true);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t bcol = tmem + lane_base + (uint32_t)(buf * dw);
      for (int c0 = 0; c0 < n_out; c0 += 16) {
        uint32_t v[16], w[16], s[16];
        tmem_ld16(bcol + c0, v);
        if (a.mma2) tmem_ld16(bcol + n_out + c0, w);
        if (bi > 0) tmem_ld16(acc_col + c0, s);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float t = __uint_as_float(v[i]);
          if (a.mma2) t += __uint_as_float(w[i]);
          s[i] = __float_as_uint(bi > 0 ? __uint_as_float(s[i]) + t : t);
        }
        tmem_st16(acc_col + c0, s);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[buf]))
                   : "memory");
    };
    // A tile of a stage arrives raw (fp32, 128B-swizzled): form hi = tf32(A)
    // in place and lo = tf32(A - hi) in the lo slot (element-wise, so the
    // swizzled layout is kept), then release the stage to the MMA warp.
    auto split_stage = [&](int st) {
      const int stage = st % stages;
      mbar_wait(&full[stage], (st / stages) & 1, false);
      float4* hi4 = reinterpret_cast<float4*>(smem + stage * stage_bytes);
      float4* lo4 = reinterpret_cast<float4*>(smem + stage * stage_bytes + a_bytes);
#pragma unroll 4
      for (int e = ct; e < (int)(a_bytes / 16); e += 128) {
        float4 v = hi4[e], h, l;
        float* pv = &v.x;
        float* ph = &h.x;
        float* pl = &l.x;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t hb, lb;
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(pv[q]));
          ph[q] = __uint_as_float(hb);
          asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(pv[q] - ph[q]));
          pl[q] = __uint_as_float(lb);
        }
        hi4[e] = h;
        lo4[e] = l;
      }
      // generic-proxy writes -> visible to the tensor core (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&ready[stage]))
                   : "memory");
    };
    int st = 0;
    for (int bi = 0; bi <= nblocks; ++bi) {
      if (a.split_smem && bi < nblocks) {
        const int vend = min(nvec, (bi + 1) * FLUSH_V);
        for (; st < vend * nchunks; ++st) split_stage(st);
      }
      if (bi >= 1) promote(bi - 1);
    }
    const int32_t tgt = a.tile_targets[slot * TMT + m];
    const int64_t ld = (int64_t)a.nsplit * n_out;
    float* o = a.acc_out + ((int64_t)(tgt < 0 ? 0 : tgt) * a.nrhs + r) * ld + (int64_t)split * n_out;
    for (int c0 = 0; c0 < n_out; c0 += 16) {
      uint32_t s[16];
      tmem_ld16(acc_col + c0, s);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (nblocks == 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) s[i] = 0u;
      }
      if (tgt >= 0) {
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(o + c0 + i) =
              make_float4(__uint_as_float(s[i]), __uint_as_float(s[i + 1]),
                          __uint_as_float(s[i + 2]), __uint_as_float(s[i + 3]));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
  }
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

// 5-D map over the dense sub-lattice array: dims (k, iz, iy, ix, p*R + r).
int make_map(CUtensorMap* tm, const float* base, int kin, int h, int64_t planes) {
  EncodeFn enc = encoder();
  if (!enc) return KIFMM_EARG;
  cuuint64_t dims[5] = {(cuuint64_t)kin, (cuuint64_t)h, (cuuint64_t)h, (cuuint64_t)h,
                        (cuuint64_t)planes};
  const cuuint64_t row = (cuuint64_t)kin * 4;
  cuuint64_t strides[4] = {row, row * h, row * h * h, row * h * h * h};
  cuuint32_t box[5] = {KC, BZ, BY, BX, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult res = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS ? 0 : KIFMM_EARG;
}

__global__ void dense_split_kernel(const float* __restrict__ qt, const int32_t* __restrict__ slot,
                                   int64_t n_boxes, int64_t nrhs, int64_t kin, int64_t h3,
                                   float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_boxes * nrhs * kin) return;
  const int64_t row = idx / kin, k = idx - row * kin;
  const int64_t b = row / nrhs, r = row - b * nrhs;
  const int32_t s = slot[b];                            // p*h3 + (ix*h + iy)*h + iz
  const int64_t p = s / h3, cell = s - p * h3;
  const int64_t d = ((p * nrhs + r) * h3 + cell) * kin + k;
  const float v = qt[idx];
  if (!lo) {                       // raw values; the sweep splits in shared memory
    hi[d] = v;
    return;
  }
  uint32_t hb;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
  const float hf = __uint_as_float(hb);
  uint32_t lb;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(v - hf));
  hi[d] = hf;
  lo[d] = __uint_as_float(lb);
}

}  // namespace

extern "C" {

// q~ rows (n_boxes*nrhs, kin) -> dense parity sub-lattice hi/lo arrays
// (8*nrhs, h, h, h, kin); rows of absent boxes are left untouched (zero).
int kifmm_dense_split_tf32(const float* qt, const int32_t* slot, int64_t n_boxes, int64_t nrhs,
                           int64_t kin, int64_t h, float* hi, float* lo, void* stream) {
  if (n_boxes < 0 || nrhs < 1 || kin < 1 || h < 1) return KIFMM_EARG;
  if (n_boxes == 0) return 0;
  const int64_t total = n_boxes * nrhs * kin;
  dense_split_kernel<<<ceil_div(total, 256), 256, 0, (cudaStream_t)stream>>>(
      qt, slot, n_boxes, nrhs, kin, h * h * h, hi, lo);
  return launch_status();
}

int kifmm_m2l_sweep_tma_f32(const float* qhi, const float* qlo, const float* bhi, const float* blo,
                            int64_t kin, int64_t n_out, int64_t h, const int32_t* tile_targets,
                            const int32_t* tile_ids, int64_t n_tiles, const int32_t* class_tv,
                            const int8_t* offsets, int64_t nrhs, int64_t nsplit, float* acc,
                            void* stream) {
  if (kin < 8 || kin % 8 || n_out < 16 || n_out > 160 || n_out % 16 ||
      n_tiles < 0 || nrhs < 1 || nsplit < 1 || nsplit > 189 || h < 1)
    return KIFMM_EARG;
  if (n_tiles == 0) return 0;
  // qlo == NULL: qhi holds the raw fp32 values and the sweep forms hi/lo in
  // shared memory (half the TMA traffic for the A operand)
  const int split_smem = qlo == nullptr;
  CUtensorMap tm_hi, tm_lo;
  int st = make_map(&tm_hi, qhi, (int)kin, (int)h, 8 * nrhs);
  if (!st) st = make_map(&tm_lo, split_smem ? qhi : qlo, (int)kin, (int)h, 8 * nrhs);
  if (st) return st;
  const size_t stage_bytes = 2 * (size_t)TMT * KC * 4 + 2 * (size_t)n_out * KC * 4;
  constexpr int max_stages = 4, ctas = 2;   // measured on B200
  // 3 * n_out accumulator columns > 256 take the whole 512-column TMEM:
  // one CTA per SM then, with the shared memory for deeper pipelining.
  // 2-MMA form (single-buffered accumulator, 3 n_out TMEM columns, two
  // CTAs/SM) where N = 2 n_out <= 256, else three MMAs per k-step.
  // Measured on B200 (config 2, level 5): ~2% faster than three MMAs; a
  // double-buffered accumulator (5 n_out columns, one CTA/SM) ~50% slower.
  constexpr int mma2_env = 2;
  const int mma2 = mma2_env && 2 * n_out <= 256 && 3 * n_out <= 256;
  const int nbuf = mma2 && mma2_env == 2 ? 1 : 2;
  const int cols = nbuf * (mma2 ? 2 : 1) * (int)n_out + (int)n_out;
  const int cps = cols > 256 ? 1 : ctas;
  int stages = (int)(((cps == 1 ? 222 * 1024 : 200 * 1024) / cps) / stage_bytes);
  if (stages > max_stages) stages = max_stages;
  if (stages < 2) return KIFMM_EARG;
  const size_t smem = 1024 + stages * stage_bytes + (3 * stages + 4) * 8 + 16;
  set_max_smem((const void*)m2l_sweep_tma_kernel, smem);
  TmaArgs a;
  a.bhi = bhi;
  a.blo = blo;
  a.kin = (int)kin;
  a.n_out = (int)n_out;
  a.stages = stages;
  a.h = (int)h;
  a.tx = (int)((h + BX - 1) / BX);
  a.ty = (int)((h + BY - 1) / BY);
  a.tz = (int)((h + BZ - 1) / BZ);
  a.tile_targets = tile_targets;
  a.tile_ids = tile_ids;
  a.class_tv = class_tv;
  a.offsets = offsets;
  a.nrhs = nrhs;
  a.nsplit = (int)nsplit;
  a.jper = (int)((189 + nsplit - 1) / nsplit);
  a.acc_out = acc;
  a.split_smem = split_smem;
  a.mma2 = mma2;
  a.nbuf = nbuf;
  dim3 grid((unsigned)n_tiles, (unsigned)nrhs, (unsigned)nsplit);
  m2l_sweep_tma_kernel<<<grid, NTHREADS, smem, (cudaStream_t)stream>>>(tm_hi, tm_lo, a);
  return launch_status();
}

}  // extern "C"
