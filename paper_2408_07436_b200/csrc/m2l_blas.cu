// BLAS-M2L fused bucket sweep (replaces the bucket loop of reference
// m2l_blas.apply_level, m2l_blas.py:284-320).
//
// The reference groups pairs by transfer vector t and, per bucket, gathers
// q~[rows_s], applies (q~ vbar_t) ubar_t^T and scatter-adds into acc[rows_t]
// (<= 316 gather/GEMM/scatter rounds, numpy-bound on the CPU).  Here the
// sweep is target-stationary: a CTA owns a tile of 128 target boxes of one
// parity class (all of which meet the same 189 transfer vectors), keeps the
// tile's accumulator in registers and streams, per vector, the gathered
// source rows and the contracted core D_t = ubar_t vbar_t^T through a
// double-buffered cp.async pipeline.  No scatter, no atomics.
//
// The 189-vector range is split into `nsplit` contiguous pieces handled by
// different CTAs (so small levels still fill the 148 SMs); each piece writes
// its own partial accumulator column block, and the expansion GEMM that
// follows (K = nsplit * ko_pad against a stacked U^T) sums them in a fixed
// order: the result is deterministic run to run.
#include "common.cuh"

using namespace kifmm;

namespace {

constexpr int TMT = 128;   // targets per tile (matches the host plan)
constexpr int RM = 4;      // accumulator rows per thread (rows tm + 32*i)
constexpr int RN = 8;      // accumulator columns per thread: RN/VEC vectors, lane-interleaved
constexpr int MAXG = 12;   // max gather chunks per thread per step (register-cached indices)

template <typename T>
struct sweep_cfg {
  static constexpr int VEC = 16 / sizeof(T);
};

template <typename T>
__global__ void __launch_bounds__(512) m2l_sweep_kernel(
    const T* __restrict__ qt, const T* __restrict__ Dt, int kin, int ko_pad, int bk,
    int nchunks, int kob, int n_slabs, int jper, const int32_t* __restrict__ tile_targets,
    const int32_t* __restrict__ tile_class, const int32_t* __restrict__ src,
    const int32_t* __restrict__ class_tv, int64_t nrhs, int nsplit, T* __restrict__ acc_out) {
  constexpr int VEC = sweep_cfg<T>::VEC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int gstride = bk + VEC;                       // padded row stride of Gs
  T* Gs = reinterpret_cast<T*>(smem_raw);             // [2][TMT][gstride]
  T* Ds = Gs + 2 * TMT * gstride;                     // [2][bk][kob]

  const int tid = threadIdx.x;
  const int nthr = blockDim.x;
  const int ng = kob / RN;
  const int tn = tid % ng, tm = tid / ng;             // tm in [0, 32)
  const int64_t tile = blockIdx.x;
  const int64_t r = blockIdx.y;
  const int slab = blockIdx.z % n_slabs, split = blockIdx.z / n_slabs;
  const int c0 = slab * kob;
  const int j0 = split * jper, j1 = min(189, j0 + jper);
  const int cls = tile_class[tile];
  const int32_t* tsrc = src + tile * 189 * TMT;       // [189][TMT]
  const int32_t* tv_list = class_tv + cls * 189;

  T acc[RM][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) acc[i][j] = T(0);

  // Staging assignment, fixed for the whole sweep: chunk e = tid + i*nthr.
  const int gch = bk / VEC;                           // 16-byte chunks per gathered row
  const int dch = kob / VEC;                          // 16-byte chunks per core row
  const int n_g = TMT * gch, n_d = bk * dch;
  int g_m[MAXG], g_off[MAXG];
#pragma unroll
  for (int i = 0; i < MAXG; ++i) {
    const int e = tid + i * nthr;
    g_m[i] = e < n_g ? e / gch : -1;
    g_off[i] = e < n_g ? (e % gch) * VEC : 0;
  }

  const int nsteps = (j1 - j0) * nchunks;
  auto stage = [&](int st, int buf) {
    const int j = j0 + st / nchunks, ch = st % nchunks;
    const int kk0 = ch * bk;
    T* g = Gs + buf * TMT * gstride;
    const int32_t* srow = tsrc + j * TMT;
#pragma unroll
    for (int i = 0; i < MAXG; ++i) {
      if (g_m[i] < 0) break;
      const int32_t s = __ldg(&srow[g_m[i]]);
      const T* gp = qt + ((int64_t)(s < 0 ? 0 : s) * nrhs + r) * kin + kk0 + g_off[i];
      cp_async16(g + g_m[i] * gstride + g_off[i], gp, s >= 0);
    }
    const T* dsrc = Dt + ((int64_t)tv_list[j] * kin + kk0) * ko_pad + c0;
    T* d = Ds + buf * bk * kob;
    for (int e = tid; e < n_d; e += nthr) {
      const int row = e / dch, v = e - row * dch;
      cp_async16(d + row * kob + v * VEC, dsrc + (int64_t)row * ko_pad + v * VEC, true);
    }
    cp_async_commit();
  };

  if (nsteps > 0) stage(0, 0);
  for (int st = 0; st < nsteps; ++st) {
    const int buf = st & 1;
    if (st + 1 < nsteps) {
      stage(st + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const T* g = Gs + buf * TMT * gstride;
    const T* d = Ds + buf * bk * kob + tn * VEC;
#pragma unroll 2
    for (int kk = 0; kk < bk; kk += VEC) {
      T a[RM][VEC];
#pragma unroll
      for (int i = 0; i < RM; ++i) {
        const T* ap = g + (tm + 32 * i) * gstride + kk;
        if constexpr (VEC == 4) {
          float4 t4 = *reinterpret_cast<const float4*>(ap);
          a[i][0] = t4.x; a[i][1] = t4.y; a[i][2] = t4.z; a[i][3] = t4.w;
        } else {
          double2 t2 = *reinterpret_cast<const double2*>(ap);
          a[i][0] = t2.x; a[i][1] = t2.y;
        }
      }
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        T b[RN];
        const T* bp = d + (kk + v) * kob;
#pragma unroll
        for (int j = 0; j < RN; j += VEC) {
          if constexpr (VEC == 4) {
            float4 t4 = *reinterpret_cast<const float4*>(bp + (j / VEC) * ng * VEC);
            b[j] = t4.x; b[j + 1] = t4.y; b[j + 2] = t4.z; b[j + 3] = t4.w;
          } else {
            double2 t2 = *reinterpret_cast<const double2*>(bp + (j / VEC) * ng * VEC);
            b[j] = t2.x; b[j + 1] = t2.y;
          }
        }
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) acc[i][j] += a[i][v] * b[j];
      }
    }
    __syncthreads();
  }

  const int64_t ld = (int64_t)nsplit * ko_pad;
#pragma unroll
  for (int i = 0; i < RM; ++i) {
    const int32_t tgt = tile_targets[tile * TMT + tm + 32 * i];
    if (tgt < 0) continue;
    T* o = acc_out + ((int64_t)tgt * nrhs + r) * ld + (int64_t)split * ko_pad + c0 + tn * VEC;
#pragma unroll
    for (int j = 0; j < RN; j += VEC) {
      T* oj = o + (j / VEC) * ng * VEC;
      if constexpr (VEC == 4) {
        *reinterpret_cast<float4*>(oj) = float4{acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]};
      } else {
        *reinterpret_cast<double2*>(oj) = double2{acc[i][j], acc[i][j + 1]};
      }
    }
  }
}

// Host-side launch geometry; must agree with device.py's blas_geometry().
template <typename T>
int sweep(const T* qt, const T* Dt, int64_t kin, int64_t ko_pad, const int32_t* tile_targets,
          const int32_t* tile_class, const int32_t* src, const int32_t* class_tv, int64_t n_tiles,
          int64_t nrhs, int64_t nsplit, T* acc, void* stream) {
  constexpr int VEC = sweep_cfg<T>::VEC;
  constexpr int BKMAX = sizeof(T) == 4 ? 64 : 32;
  if (kin < VEC || ko_pad < RN || n_tiles < 0 || nrhs < 1 || nsplit < 1 || nsplit > 189)
    return KIFMM_EARG;
  if (kin % VEC || ko_pad % RN) return KIFMM_EARG;
  if (n_tiles == 0) return 0;
  const int nchunks = (int)((kin + BKMAX - 1) / BKMAX);
  if (kin % nchunks) return KIFMM_EARG;
  const int bk = (int)(kin / nchunks);
  if (bk % VEC) return KIFMM_EARG;
  const int n_slabs = (int)((ko_pad + 127) / 128);
  if (ko_pad % n_slabs) return KIFMM_EARG;
  const int kob = (int)(ko_pad / n_slabs);
  if (kob % RN) return KIFMM_EARG;
  const int threads = 32 * (kob / RN);
  if ((TMT * (bk / VEC) + threads - 1) / threads > MAXG) return KIFMM_EARG;
  const int jper = (int)((189 + nsplit - 1) / nsplit);
  const size_t smem = sizeof(T) * (2 * TMT * (bk + VEC) + 2 * bk * kob);
  auto kern = m2l_sweep_kernel<T>;
  set_max_smem((const void*)kern, smem);
  dim3 grid((unsigned)n_tiles, (unsigned)nrhs, (unsigned)(n_slabs * nsplit));
  kern<<<grid, threads, smem, (cudaStream_t)stream>>>(qt, Dt, (int)kin, (int)ko_pad, bk, nchunks,
                                                      kob, n_slabs, jper, tile_targets,
                                                      tile_class, src, class_tv, nrhs,
                                                      (int)nsplit, acc);
  return launch_status();
}

// ---------------------------------------------------------------------------
// FP64 sweep on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64): same
// target-stationary structure, but each warp owns a 32 x (kob/2) block of
// the tile's accumulator as 4 x NTW m8n8 fragments, and every k4 step is
// 4 + NTW fragment loads for 4 * NTW DMMAs (256 FMAs each) -- the FP64
// pipe, not instruction issue or shared memory, sets the pace.  Exact IEEE
// fp64 products and sums (only the summation order differs from SIMT).
// Geometry (device.py blas_geometry): kin % 16 == 0; ko_pad = n_slabs * kob,
// kob % 16 == 0, kob <= 160, n_slabs = ceil(ko_pad / 160).
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int NTW, int BKT, int STG, int MINB>
__global__ void __launch_bounds__(256, MINB) m2l_sweep_dmma_kernel(
    const double* __restrict__ qt, const double* __restrict__ Dt, int kin, int ko_pad,
    int nchunks, int n_slabs, int jper, const int32_t* __restrict__ tile_targets,
    const int32_t* __restrict__ tile_class, const int32_t* __restrict__ src,
    const int32_t* __restrict__ class_tv, int64_t nrhs, int nsplit,
    const uint16_t* __restrict__ gmask, const int16_t* __restrict__ jlist,
    const int32_t* __restrict__ jcount, double* __restrict__ acc_out) {
  constexpr int BK = BKT;                             // k-chunk per pipeline stage
  constexpr int GS = BK + 4;                          // row stride = 32 mod 128 bytes: conflict-free A
  constexpr int KOB = 16 * NTW;
  constexpr int DS = KOB + 4;                         // Ds row stride = 4 mod 16 doubles: the 16 lanes of a
                                                      // half-warp (rows lane & 3, columns lane >> 2) hit 16
                                                      // distinct 8-byte bank pairs (KOB + 8: rows k, k + 2 collide)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Gs = reinterpret_cast<double*>(smem_raw);   // [STG][TMT][GS]
  double* Ds = Gs + STG * TMT * GS;                   // [STG][BK][DS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;
  const int64_t tile = blockIdx.x;
  const int64_t r = blockIdx.y;
  const int slab = blockIdx.z % n_slabs, split = blockIdx.z / n_slabs;
  const int c0 = slab * KOB;
  // Sparse trees: the tile's vectors with at least one source (jlist, in
  // ascending order) are split over the CTAs of the tile, and per vector the
  // 8-row groups without any source (gmask bit clear) skip their DMMAs.
  const int cnt = jcount ? jcount[tile] : 189;
  const int jp = jcount ? (cnt + nsplit - 1) / nsplit : jper;
  const int j0 = split * jp, j1 = min(cnt, j0 + jp);
  const int16_t* jl = jlist ? jlist + tile * 189 : nullptr;
  const uint16_t* gm = gmask ? gmask + tile * 189 : nullptr;
  auto vec_of = [&](int p) { return jl ? (int)jl[p] : p; };
  __shared__ uint32_t stage_bits[STG];
  const int32_t* tsrc = src + tile * 189 * TMT;
  const int32_t* tv_list = class_tv + tile_class[tile] * 189;

  double acc[4][NTW][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NTW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // Gather assignment: 16-byte chunk tid % CPR of rows tid / CPR + RPP * i.
  constexpr int CPR = BK / 2, RPP = 256 / CPR, NR = TMT / RPP;
  const int grow = tid / CPR, gch = tid % CPR;
  int ids_cur[NR], ids_next[NR];
  auto load_ids = [&](int j, int (&ids)[NR]) {
#pragma unroll
    for (int i = 0; i < NR; ++i)
      ids[i] = j < j1 ? __ldg(&tsrc[vec_of(j) * TMT + grow + RPP * i]) : -1;
  };
  const int nsteps = (j1 - j0) * nchunks;
  auto stage = [&](int st, int buf) {
    const int p = j0 + st / nchunks, ch = st % nchunks;
    const int j = vec_of(p);
    if (ch == 0) {
#pragma unroll
      for (int i = 0; i < NR; ++i) ids_cur[i] = ids_next[i];
      load_ids(p + 1, ids_next);
    }
    if (tid == 0) stage_bits[buf] = gm ? (uint32_t)gm[j] : 0xFFFFu;
    const int kk0 = ch * BK;
    const bool kin_ok = kk0 + 2 * gch < kin;           // a partial last chunk reads zeros
    double* g = Gs + buf * TMT * GS;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int s = ids_cur[i];
      const bool ok = s >= 0 && kin_ok;
      const double* gp = qt + ((int64_t)(ok ? s : 0) * nrhs + r) * kin + (ok ? kk0 + 2 * gch : 0);
      cp_async16(g + (grow + RPP * i) * GS + 2 * gch, gp, ok);
    }
    const double* dsrc = Dt + ((int64_t)tv_list[j] * kin + kk0) * ko_pad + c0;
    double* d = Ds + buf * BK * DS;
    constexpr int DCH = BK * KOB / 2;
    for (int e = tid; e < DCH; e += 256) {
      const int row = e / (KOB / 2), v = e - row * (KOB / 2);
      const bool ok = kk0 + row < kin;
      cp_async16(d + row * DS + 2 * v, ok ? dsrc + (int64_t)row * ko_pad + 2 * v : Dt, ok);
    }
    cp_async_commit();
  };

  load_ids(j0, ids_next);
  // STG-deep cp.async ring: stages st+1 .. st+STG-1 in flight while st computes
  for (int q = 0; q < STG - 1; ++q) {
    if (q < nsteps) stage(q, q);
    else cp_async_commit();
  }
  const int arow = 32 * wm + (lane >> 2), acol = lane & 3;
  const int bcol = wn * (KOB / 2) + (lane >> 2), brow = lane & 3;
  for (int st = 0; st < nsteps; ++st) {
    const int buf = st % STG;
    cp_async_wait<STG - 2>();
    __syncthreads();
    if (st + STG - 1 < nsteps) stage(st + STG - 1, (st + STG - 1) % STG);
    else cp_async_commit();
    const double* g = Gs + buf * TMT * GS + arow * GS + acol;
    const double* d = Ds + buf * BK * DS + brow * DS + bcol;
    const uint32_t mb = (stage_bits[buf] >> (4 * wm)) & 0xFu;   // warp-uniform
    if (mb == 0xFu) {
#pragma unroll
      for (int ks = 0; ks < BK; ks += 4) {
        double a[4], b[NTW];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) a[mt] = g[mt * 8 * GS + ks];
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt) b[nt] = d[ks * DS + nt * 8];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) dmma884(acc[mt][nt], a[mt], b[nt]);
      }
    } else if (mb) {
#pragma unroll 2
      for (int ks = 0; ks < BK; ks += 4) {
        double b[NTW];
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt) b[nt] = d[ks * DS + nt * 8];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          if (!((mb >> mt) & 1u)) continue;
          const double a = g[mt * 8 * GS + ks];
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) dmma884(acc[mt][nt], a, b[nt]);
        }
      }
    }
  }
  cp_async_wait<0>();

  const int64_t ld = (int64_t)nsplit * ko_pad;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int32_t tgt = tile_targets[tile * TMT + 32 * wm + 8 * mt + (lane >> 2)];
    if (tgt < 0) continue;
    double* o = acc_out + ((int64_t)tgt * nrhs + r) * ld + (int64_t)split * ko_pad + c0 +
                wn * (KOB / 2) + 2 * (lane & 3);
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt)
      *reinterpret_cast<double2*>(o + nt * 8) = double2{acc[mt][nt][0], acc[mt][nt][1]};
  }
}

int sweep_dmma(const double* qt, const double* Dt, int64_t kin, int64_t ko_pad,
               const int32_t* tile_targets, const int32_t* tile_class, const int32_t* src,
               const int32_t* class_tv, int64_t n_tiles, int64_t nrhs, int64_t nsplit,
               const uint16_t* gmask, const int16_t* jlist, const int32_t* jcount, double* acc,
               void* stream) {
  constexpr int KOB_MAX = 160;
  if (kin < 16 || kin % 16 || ko_pad < 16 || n_tiles < 0 || nrhs < 1 || nsplit < 1 ||
      nsplit > 189)
    return KIFMM_EARG;
  if (n_tiles == 0) return 0;
  const int n_slabs = (int)((ko_pad + KOB_MAX - 1) / KOB_MAX);
  if (ko_pad % n_slabs) return KIFMM_EARG;
  const int kob = (int)(ko_pad / n_slabs);
  if (kob % 16 || kob > KOB_MAX) return KIFMM_EARG;
  const int jper = (int)((189 + nsplit - 1) / nsplit);
  dim3 grid((unsigned)n_tiles, (unsigned)nrhs, (unsigned)(n_slabs * nsplit));
  cudaStream_t s = (cudaStream_t)stream;
  // Pipeline: 32-wide K chunks, 3 stages for large ranks (many stages per
  // vector; latency-bound at 2 x 16); 16-wide double buffering for small k.
  const bool wide = kin >= 64;
  const int bk = wide ? 32 : 16;
  const int nchunks = (int)((kin + bk - 1) / bk);
  auto smem_of = [&](int st) {
    return sizeof(double) * (size_t)st * (TMT * (bk + 4) + bk * (kob + 4));
  };
  const int stg = (wide && smem_of(3) <= 227 * 1024) ? 3 : 2;
  const size_t smem = smem_of(stg);
#define KIFMM_DMMA(NT_, BK_, STG_, MB_)                                                         \
  {                                                                                              \
    auto k_ = m2l_sweep_dmma_kernel<NT_, BK_, STG_, MB_>;                                        \
    set_max_smem((const void*)k_, smem);                                                         \
    k_<<<grid, 256, smem, s>>>(qt, Dt, (int)kin, (int)ko_pad, nchunks, n_slabs, jper,            \
                               tile_targets, tile_class, src, class_tv, nrhs, (int)nsplit,       \
                               gmask, jlist, jcount, acc);                                       \
  }
#define KIFMM_DMMA_NT(NT_)                                                                      \
  case NT_:                                                                                      \
    if (wide && stg == 3) KIFMM_DMMA(NT_, 32, 3, 1)                                              \
    else if (wide) KIFMM_DMMA(NT_, 32, 2, 1)                                                     \
    else KIFMM_DMMA(NT_, 16, 2, (NT_ > 5 ? 1 : 2))                                               \
    break;
  switch (kob / 16) {
    KIFMM_DMMA_NT(1) KIFMM_DMMA_NT(2) KIFMM_DMMA_NT(3) KIFMM_DMMA_NT(4) KIFMM_DMMA_NT(5)
    KIFMM_DMMA_NT(6) KIFMM_DMMA_NT(7) KIFMM_DMMA_NT(8) KIFMM_DMMA_NT(9) KIFMM_DMMA_NT(10)
    default:
      return KIFMM_EARG;
  }
#undef KIFMM_DMMA_NT
#undef KIFMM_DMMA
  return launch_status();
}

}  // namespace

extern "C" {

int kifmm_m2l_sweep_f32(const float* qt, const float* Dt, int64_t kin, int64_t ko_pad,
                        const int32_t* tile_targets, const int32_t* tile_class, const int32_t* src,
                        const int32_t* class_tv, int64_t n_tiles, int64_t nrhs, int64_t nsplit,
                        float* acc, void* s) {
  return sweep<float>(qt, Dt, kin, ko_pad, tile_targets, tile_class, src, class_tv, n_tiles, nrhs,
                      nsplit, acc, s);
}
int kifmm_m2l_sweep_f64(const double* qt, const double* Dt, int64_t kin, int64_t ko_pad,
                        const int32_t* tile_targets, const int32_t* tile_class, const int32_t* src,
                        const int32_t* class_tv, int64_t n_tiles, int64_t nrhs, int64_t nsplit,
                        double* acc, void* s) {
  return sweep_dmma(qt, Dt, kin, ko_pad, tile_targets, tile_class, src, class_tv, n_tiles, nrhs,
                    nsplit, nullptr, nullptr, nullptr, acc, s);
}
int kifmm_m2l_sweep_sparse_f64(const double* qt, const double* Dt, int64_t kin, int64_t ko_pad,
                               const int32_t* tile_targets, const int32_t* tile_class,
                               const int32_t* src, const int32_t* class_tv, int64_t n_tiles,
                               int64_t nrhs, int64_t nsplit, const uint16_t* gmask,
                               const int16_t* jlist, const int32_t* jcount, double* acc,
                               void* s) {
  if (!gmask || !jlist || !jcount) return KIFMM_EARG;
  return sweep_dmma(qt, Dt, kin, ko_pad, tile_targets, tile_class, src, class_tv, n_tiles, nrhs,
                    nsplit, gmask, jlist, jcount, acc, s);
}

}  // extern "C"
