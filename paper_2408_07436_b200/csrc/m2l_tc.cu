// BLAS-M2L fused sweep on the 5th-generation tensor cores (tcgen05, sm_100a),
// float32 path via 3xTF32 splitting.
//
// Same contraction as m2l_blas.cu (target-stationary, one CTA per tile of
// 128 same-parity target boxes, 189 transfer vectors in ascending order,
// optional split of the vector range into pieces with partial accumulators),
// but the (128 x k) . (k x N) product per vector runs as
//     acc += A_lo B_hi + A_hi B_lo + A_hi B_hi
// with A = gathered source rows of q~ and B = the dense core D_t, both split
// into a TF32 "hi" part and a TF32 residual "lo" part, so the result keeps
// ~fp32 accuracy (the TF32 products themselves would lose ~3 digits).
//
// Roles (288 threads):
//   warps 0-3  producers: thread m gathers row m of A_hi/A_lo with cp.async
//              into the canonical K-major no-swizzle layout (8-row x 16-byte
//              core matrices) and copies its share of the pre-laid-out
//              B_hi/B_lo block; completion is tracked on the stage's "full"
//              mbarrier (cp.async.mbarrier.arrive.noinc).
//   warp 4     allocates TMEM (two 128 x N fp32 MMA buffers + one long-lived
//              accumulator) and one elected thread issues
//              tcgen05.mma.kind::tf32, releasing each stage with
//              tcgen05.commit -> "empty" mbarrier.
//   warps 5-8  accumulators/epilogue: every FLUSH_V vectors they add the
//              finished MMA buffer into the long-lived accumulator with IEEE
//              fp32 adds (tcgen05.ld / tcgen05.st), then write the result.
#include <cstdlib>

#include "common.cuh"

using namespace kifmm;

namespace {

constexpr int TMT = 128;        // targets per tile = MMA M
constexpr int KC = 32;          // K (floats) per pipeline stage
constexpr int NPROD = 128;      // producer threads
constexpr int NTHREADS = 288;   // 4 producer + 1 MMA + 4 accumulator warps

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  uint32_t spins = 0;
  while (!done) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (!done && ++spins > (1u << 26)) __trap();   // watchdog: a lost arrive faults, never hangs
  }
}

// Wait for non-latency-critical roles: back off with nanosleep so the
// spinning warp does not steal issue slots from the producers sharing its
// SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  uint32_t spins = 0;
  while (true) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(256);
    if (++spins > (1u << 24)) __trap();
  }
}

__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Shared-memory matrix descriptor, SWIZZLE_NONE, K-major canonical layout:
// core matrices of 8 rows x 16 bytes; LBO = byte stride between core matrices
// along K, SBO = byte stride between 8-row groups along M/N.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;                       // descriptor version (sm_100)
  return d;                                     // base offset 0, layout SWIZZLE_NONE
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

// TMEM accumulation is periodically promoted: the MMA accumulates FLUSH_V
// vectors into one of two TMEM buffers, then the accumulator warps add that
// buffer into a long-lived TMEM region with IEEE fp32 adds (tensor-core
// accumulation over the ~3*189*k products of a full sweep loses ~1e-5).
constexpr int FLUSH_V = 4;

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

__global__ void __launch_bounds__(NTHREADS) m2l_sweep_tc_kernel(
    const float* __restrict__ qhi, const float* __restrict__ qlo, const float* __restrict__ bhi,
    const float* __restrict__ blo, int kin, int n_out, int stages,
    const int32_t* __restrict__ tile_targets, const int32_t* __restrict__ tile_class,
    const int32_t* __restrict__ src, const int32_t* __restrict__ class_tv, int64_t nrhs,
    int nsplit, int jper, int l1_gather, float* __restrict__ acc_out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nchunks = (kin + KC - 1) / KC;
  const uint32_t a_bytes = TMT * KC * 4;                 // 16 KB
  const uint32_t b_bytes = (uint32_t)n_out * KC * 4;
  const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;                      // [2] MMA -> accumulators
  uint64_t* tempty = tfull + 2;                          // [2] accumulators -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int64_t tile = blockIdx.x;
  const int64_t r = blockIdx.y;
  const int split = blockIdx.z;
  const int j0 = split * jper, j1 = min(189, j0 + jper);
  const int nvec = max(0, j1 - j0);
  const int nsteps = nvec * nchunks;
  const int nblocks = (nvec + FLUSH_V - 1) / FLUSH_V;
  const int cls = tile_class[tile];
  const int32_t* tsrc = src + tile * 189 * TMT;
  const int32_t* tv_list = class_tv + cls * 189;
  // columns: [0, n) and [n, 2n) MMA buffers, [2n, 3n) long-lived accumulator
  const uint32_t need = 3u * (uint32_t)n_out;
  const uint32_t tmem_cols = need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : need <= 256 ? 256 : 512;

  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], NPROD + 1);   // 128 cp.async arrivals + the bulk-copy expect_tx
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tfull[1], 1);
    mbar_init(&tempty[0], NPROD);
    mbar_init(&tempty[1], NPROD);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ------------------------------------------------------------ producers
    // Warp w gathers rows [32w, 32w+32).  Lane l owns the source index of row
    // 32w+l (prefetched one vector ahead); the copies go 8 lanes per row, so
    // one instruction moves 4 full 128-byte row segments (whole sectors).
    const int sub_row = lane >> 3, sub_ch = lane & 7;
    int32_t s_cur = nvec > 0 ? __ldg(&tsrc[j0 * TMT + tid]) : -1;
    int32_t s_next = nvec > 1 ? __ldg(&tsrc[(j0 + 1) * TMT + tid]) : -1;
    for (int st = 0; st < nsteps; ++st) {
      const int stage = st % stages;
      const int round = st / stages;
      if (round > 0) mbar_wait(&empty[stage], (round - 1) & 1);
      const int jl = st / nchunks, c = st % nchunks;
      const int j = j0 + jl;
      if (c == 0 && jl > 0) {
        s_cur = s_next;
        s_next = jl + 1 < nvec ? __ldg(&tsrc[(j + 1) * TMT + tid]) : -1;
      }
      const int kc = min(KC, kin - c * KC);              // multiple of 8
      unsigned char* sb = smem + stage * stage_bytes;
      if (tid == 0) {
        // B block of (vector, chunk): already in smem layout, contiguous.
        const uint32_t bbytes = (uint32_t)(n_out * kc * 4);
        const int64_t boff = (int64_t)tv_list[j] * n_out * kin + (int64_t)n_out * KC * c;
        const uint32_t fb = smem_u32(&full[stage]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb),
                     "r"(2 * bbytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sb + 2 * a_bytes)),
            "l"(bhi + boff), "r"(bbytes), "r"(fb)
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sb + 2 * a_bytes + b_bytes)),
            "l"(blo + boff), "r"(bbytes), "r"(fb)
            : "memory");
      }
      const bool ch_live = sub_ch < kc / 4;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rl = i * 4 + sub_row;                  // row within the warp's 32
        const int32_t s = __shfl_sync(0xffffffffu, s_cur, rl);
        if (ch_live) {
          const int m = warp * 32 + rl;
          const uint32_t off = (m >> 3) * (KC / 4) * 128 + (m & 7) * 16 + sub_ch * 128;
          const int64_t g = ((int64_t)(s < 0 ? 0 : s) * nrhs + r) * kin + c * KC + sub_ch * 4;
          if (l1_gather) {
            cp_async16_ca(sb + off, qhi + g, s >= 0);
            cp_async16_ca(sb + a_bytes + off, qlo + g, s >= 0);
          } else {
            cp_async16(sb + off, qhi + g, s >= 0);
            cp_async16(sb + a_bytes + off, qlo + g, s >= 0);
          }
        }
      }
      cp_async_arrive_noinc(&full[stage]);
    }
  } else if (warp == 4) {
    // ----------------------------------------------------------- MMA issue
    // idesc: D f32 (bit 4), A/B tf32 (bits 7, 10), K-major A and B,
    // N >> 3 at bit 17, M >> 4 at bit 24.
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n_out >> 3) << 17) |
                           ((uint32_t)(TMT >> 4) << 24);
    if (lane == 0) {
      int st = 0;
      for (int bi = 0; bi < nblocks; ++bi) {
        const int buf = bi & 1;
        if (bi >= 2) mbar_wait(&tempty[buf], ((bi >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dcol = tmem + (uint32_t)(buf * n_out);
        const int vend = min(nvec, (bi + 1) * FLUSH_V);
        uint32_t acc_flag = 0;
        for (; st < vend * nchunks; ++st) {
          const int stage = st % stages;
          mbar_wait(&full[stage], (st / stages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const int c = st % nchunks;
          const int kc = min(KC, kin - c * KC);
          const uint32_t base = smem_u32(smem + stage * stage_bytes);
          const uint32_t a_hi = base, a_lo = base + a_bytes;
          const uint32_t b_hi = base + 2 * a_bytes, b_lo = b_hi + b_bytes;
          const uint32_t sbo_a = (KC / 4) * 128, sbo_b = (uint32_t)(kc / 4) * 128;
          for (int ks = 0; ks < kc / 8; ++ks) {
            const uint32_t ko = ks * 256;
            mma_tf32(dcol, smem_desc(a_lo + ko, 128, sbo_a), smem_desc(b_hi + ko, 128, sbo_b),
                     idesc, acc_flag);
            acc_flag = 1;
            mma_tf32(dcol, smem_desc(a_hi + ko, 128, sbo_a), smem_desc(b_lo + ko, 128, sbo_b),
                     idesc, 1);
            mma_tf32(dcol, smem_desc(a_hi + ko, 128, sbo_a), smem_desc(b_hi + ko, 128, sbo_b),
                     idesc, 1);
          }
          mma_commit(&empty[stage]);
        }
        mma_commit(&tfull[buf]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------- accumulator warps (5..8) + epilogue
    const int sub = warp & 3;                            // TMEM sub-partition of this warp
    const int m = sub * 32 + lane;                       // accumulator row = target slot
    const uint32_t lane_base = (uint32_t)(sub * 32) << 16;
    const uint32_t acc_col = tmem + lane_base + 2u * (uint32_t)n_out;
    for (int bi = 0; bi < nblocks; ++bi) {
      const int buf = bi & 1;
      mbar_wait_sleep(&tfull[buf], (bi >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t bcol = tmem + lane_base + (uint32_t)(buf * n_out);
      for (int c0 = 0; c0 < n_out; c0 += 16) {
        uint32_t v[16], a[16];
        tmem_ld16(bcol + c0, v);
        if (bi > 0) tmem_ld16(acc_col + c0, a);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; ++i)
          a[i] = bi > 0 ? __float_as_uint(__uint_as_float(a[i]) + __uint_as_float(v[i])) : v[i];
        tmem_st16(acc_col + c0, a);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[buf]))
                   : "memory");
    }
    const int32_t tgt = tile_targets[tile * TMT + m];
    const int64_t ld = (int64_t)nsplit * n_out;
    float* o = acc_out + ((int64_t)(tgt < 0 ? 0 : tgt) * nrhs + r) * ld + (int64_t)split * n_out;
    for (int c0 = 0; c0 < n_out; c0 += 16) {
      uint32_t a[16];
      tmem_ld16(acc_col + c0, a);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (nblocks == 0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = 0u;          // empty piece: zero partial
      }
      if (tgt >= 0) {
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(o + c0 + i) =
              make_float4(__uint_as_float(a[i]), __uint_as_float(a[i + 1]),
                          __uint_as_float(a[i + 2]), __uint_as_float(a[i + 3]));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 4) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
  }
}

__global__ void split_tf32_kernel(const float* __restrict__ x, int64_t n, float* __restrict__ hi,
                                  float* __restrict__ lo) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float v = x[i];
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
  const float hf = __uint_as_float(h);
  uint32_t l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(v - hf));
  hi[i] = hf;
  lo[i] = __uint_as_float(l);
}

}  // namespace

extern "C" {

// hi/lo TF32 split of a float32 array (x = hi + lo + O(2^-22 |x|)).
int kifmm_split_tf32(const float* x, int64_t n, float* hi, float* lo, void* stream) {
  if (n < 0) return KIFMM_EARG;
  if (n == 0) return 0;
  split_tf32_kernel<<<ceil_div(n, 256), 256, 0, (cudaStream_t)stream>>>(x, n, hi, lo);
  return launch_status();
}

int kifmm_m2l_sweep_tc_f32(const float* qhi, const float* qlo, const float* bhi, const float* blo,
                           int64_t kin, int64_t n_out, const int32_t* tile_targets,
                           const int32_t* tile_class, const int32_t* src, const int32_t* class_tv,
                           int64_t n_tiles, int64_t nrhs, int64_t nsplit, float* acc, void* stream) {
  if (kin < 8 || kin % 8 || n_out < 16 || n_out > 160 || n_out % 16 || n_tiles < 0 || nrhs < 1 ||
      nsplit < 1 || nsplit > 189)
    return KIFMM_EARG;
  if (n_tiles == 0) return 0;
  const size_t stage_bytes = 2 * (size_t)TMT * KC * 4 + 2 * (size_t)n_out * KC * 4;
  // Pipeline depth / CTAs per SM (measured on B200)
  constexpr int ctas_per_sm = 2, max_stages = 6, l1 = 0;
  // 3 * n_out accumulator columns > 256 take the whole 512-column TMEM:
  // one CTA per SM then (a second one would wait in tcgen05.alloc).
  const int ctas = 3 * n_out > 256 ? 1 : ctas_per_sm;
  int stages = (int)((220 * 1024 / ctas) / stage_bytes);
  if (stages > max_stages) stages = max_stages;
  if (stages < 2) return KIFMM_EARG;
  const size_t smem = stages * stage_bytes + (2 * stages + 4) * 8 + 16;
  const int jper = (int)((189 + nsplit - 1) / nsplit);
  set_max_smem((const void*)m2l_sweep_tc_kernel, smem);
  dim3 grid((unsigned)n_tiles, (unsigned)nrhs, (unsigned)nsplit);
  m2l_sweep_tc_kernel<<<grid, NTHREADS, smem, (cudaStream_t)stream>>>(
      qhi, qlo, bhi, blo, (int)kin, (int)n_out, stages, tile_targets, tile_class, src, class_tv,
      nrhs, (int)nsplit, jper, l1, acc);
  return launch_status();
}

}  // extern "C"
