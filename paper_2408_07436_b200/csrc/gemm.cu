// Tall-skinny SIMT GEMM for the level operators (projection/expansion of
// BLAS-M2L, factored pseudo-inverse solves, M2M/L2L kernel products).
// These are memory/latency-bound (N, K <= a few hundred, M up to 2M rows),
// so a register-tiled FFMA/DFMA kernel with shared-memory staging and a
// register prefetch of the next K-tile is enough.  The epilogue fuses the
// pseudo-inverse's diagonal (colscale), the level scale (alpha),
// accumulation and the L2L child scatter (rowmap).  The A loader can sum
// `asum` column blocks (stride `astride`): that is how the partial
// accumulators of the split M2L sweep are reduced, in a fixed order.
#include <cstdlib>

#include "common.cuh"

using namespace kifmm;

namespace {

constexpr int BN = 64, BK = 16, TN = 4, NT = 256;

template <typename T, int BM>
__global__ void __launch_bounds__(NT) gemm_kernel(int64_t M, int64_t N, int64_t K, T alpha,
                                                  const T* __restrict__ A, int64_t lda,
                                                  int asum, int64_t astride,
                                                  const T* __restrict__ B, int64_t ldb,
                                                  const T* __restrict__ colscale,
                                                  T* __restrict__ C, int64_t ldc,
                                                  const int32_t* __restrict__ rowmap,
                                                  int accumulate) {
  constexpr int TM = BM * BN / (NT * TN);        // rows per thread: 4 (BM=64), 2, 1
  constexpr int AE = BM * BK / NT;               // A elements loaded per thread
  constexpr int BE = BK * BN / NT;               // B elements loaded per thread (4)
  __shared__ __align__(16) T As[BK][BM + 4];
  __shared__ __align__(16) T Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tn = tid % (BN / TN), tm = tid / (BN / TN);
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

  T ra[AE], rb[BE];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int e = 0; e < AE; ++e) {
      const int idx = tid + e * NT;
      const int r = idx / BK, c = idx % BK;
      const int64_t gm = m0 + r, gk = k0 + c;
      T v = T(0);
      if (gm < M && gk < K) {
        const T* p = A + gm * lda + gk;
        v = p[0];
        for (int s = 1; s < asum; ++s) v += p[s * astride];
      }
      ra[e] = v;
    }
#pragma unroll
    for (int e = 0; e < BE; ++e) {
      const int idx = tid + e * NT;
      const int r = idx / BN, c = idx % BN;
      const int64_t gk = k0 + r, gn = n0 + c;
      rb[e] = (gk < K && gn < N) ? B[gk * ldb + gn] : T(0);
    }
  };
  load(0);
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int e = 0; e < AE; ++e) {
      const int idx = tid + e * NT;
      As[idx % BK][idx / BK] = ra[e];
    }
#pragma unroll
    for (int e = 0; e < BE; ++e) {
      const int idx = tid + e * NT;
      Bs[idx / BN][idx % BN] = rb[e];
    }
    __syncthreads();
    if (k0 + BK < K) load(k0 + BK);              // overlap the next tile's loads
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      // vector shared loads: the TM rows and TN columns of a thread are
      // contiguous (one 16-byte load each for float; TM may be 1 or 2)
      T a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][tm * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tn * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] += a[i] * b[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t gm = m0 + tm * TM + i;
    if (gm >= M) continue;
    const int64_t row = rowmap ? (int64_t)rowmap[gm] : gm;
    if (row < 0) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t gn = n0 + tn * TN + j;
      if (gn >= N) continue;
      T v = acc[i][j];
      if (colscale) v *= colscale[gn];
      v *= alpha;
      T* dst = C + row * ldc + gn;
      *dst = accumulate ? *dst + v : v;
    }
  }
}

template <typename T, int BM>
int launch_gemm(int64_t M, int64_t N, int64_t K, T alpha, const T* A, int64_t lda, int asum,
                int64_t astride, const T* B, int64_t ldb, const T* colscale, T* C, int64_t ldc,
                const int32_t* rowmap, int accumulate, cudaStream_t s) {
  const int64_t max_rows = (int64_t)65535 * BM;
  for (int64_t r0 = 0; r0 < M; r0 += max_rows) {
    const int64_t mm = M - r0 < max_rows ? M - r0 : max_rows;
    dim3 grid(ceil_div(N, BN), ceil_div(mm, BM));
    gemm_kernel<T, BM><<<grid, NT, 0, s>>>(mm, N, K, alpha, A + r0 * lda, lda, asum, astride, B,
                                           ldb, colscale, rowmap ? C : C + r0 * ldc, ldc,
                                           rowmap ? rowmap + r0 : nullptr, accumulate);
  }
  return launch_status();
}

template <typename T>
int gemm(int64_t M, int64_t N, int64_t K, T alpha, const T* A, int64_t lda, int asum,
         int64_t astride, const T* B, int64_t ldb, const T* colscale, T* C, int64_t ldc,
         const int32_t* rowmap, int accumulate, void* stream) {
  if (M < 0 || N < 0 || K < 0 || asum < 1) return KIFMM_EARG;
  if (M == 0 || N == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  // Pick the row tile so that the grid covers the 148 SMs when possible.
  const int64_t ncol = (N + BN - 1) / BN;
  if (M * ncol >= 64 * 148 * 2)
    return launch_gemm<T, 64>(M, N, K, alpha, A, lda, asum, astride, B, ldb, colscale, C, ldc,
                              rowmap, accumulate, s);
  if (M * ncol >= 32 * 148)
    return launch_gemm<T, 32>(M, N, K, alpha, A, lda, asum, astride, B, ldb, colscale, C, ldc,
                              rowmap, accumulate, s);
  return launch_gemm<T, 16>(M, N, K, alpha, A, lda, asum, astride, B, ldb, colscale, C, ldc,
                            rowmap, accumulate, s);
}

// ---------------------------------------------------------------------------
// float32 tall-skinny GEMM, the throughput form used for >= 4k-row operator
// applications: CTA tile 128 x 64, 256 threads of 8 x 4 outputs, 16-deep K
// stages double-buffered in shared memory.  A rows and B rows arrive by
// 16-byte cp.async when aligned (one instruction per 16 bytes, no register
// staging); the split-sum A loader (asum > 1) and unaligned shapes go through
// registers.  Same contract (colscale, alpha, accumulate, row scatter) as
// gemm_kernel.  The per-thread 8 A values are broadcast loads (a warp spans
// two row groups), the 4 B values one 16-byte load.
constexpr int SBM = 128, SBN = 64, SBK = 16;
constexpr int SAS = SBK + 4;      // A tile row stride (floats): 16-byte rows, rows on distinct banks
constexpr int SBS = SBN + 4;      // B tile row stride

__global__ void __launch_bounds__(256) gemm_ts_kernel(
    int64_t M, int64_t N, int64_t K, float alpha, const float* __restrict__ A, int64_t lda,
    int asum, int64_t astride, const float* __restrict__ B, int64_t ldb,
    const float* __restrict__ colscale, float* __restrict__ C, int64_t ldc,
    const int32_t* __restrict__ rowmap, int accumulate, int async_a, int async_b) {
  __shared__ __align__(16) float As[2][SBM * SAS];
  __shared__ __align__(16) float Bs[2][SBK * SBS];
  const int tid = threadIdx.x;
  const int tn = tid & 15, tm = tid >> 4;         // 16 column groups of 4, 16 row groups of 8
  const int64_t m0 = (int64_t)blockIdx.y * SBM, n0 = (int64_t)blockIdx.x * SBN;
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  auto stage = [&](int64_t k0, int buf) {
    // A: 128 rows x 4 chunks of 4 floats
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int e = tid + it * 256;
      const int r = e >> 2, c = (e & 3) * 4;
      const int64_t gm = m0 + r, gk = k0 + c;
      float* dst = &As[buf][r * SAS + c];
      if (async_a) {
        const bool ok = gm < M && gk < K;         // K % 4 == 0: the chunk is in or out
        cp_async16(dst, ok ? A + gm * lda + gk : A, ok);
      } else {
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (gm < M) {
          const float* p = A + gm * lda;
          for (int q = 0; q < asum; ++q)
#pragma unroll
            for (int h = 0; h < 4; ++h)
              if (gk + h < K) v[h] += p[q * astride + gk + h];
        }
        *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
    // B: 16 rows x 16 chunks of 4 floats
    {
      const int e = tid;
      const int r = e >> 4, c = (e & 15) * 4;
      const int64_t gk = k0 + r, gn = n0 + c;
      float* dst = &Bs[buf][r * SBS + c];
      if (async_b) {
        const bool ok = gk < K && gn < N;         // N % 4 == 0
        cp_async16(dst, ok ? B + gk * ldb + gn : B, ok);
      } else {
        float v[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) v[h] = (gk < K && gn + h < N) ? B[gk * ldb + gn + h] : 0.f;
        *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
    cp_async_commit();
  };

  const int nk = (int)((K + SBK - 1) / SBK);
  stage(0, 0);
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) {
      stage((int64_t)(kt + 1) * SBK, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float* a = &As[buf][(tm * 8) * SAS];
    const float* b = &Bs[buf][tn * 4];
#pragma unroll
    for (int kk = 0; kk < SBK; ++kk) {
      const float4 bv = *reinterpret_cast<const float4*>(b + kk * SBS);
      float av[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) av[i] = a[i * SAS + kk];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        acc[i][0] = fmaf(av[i], bv.x, acc[i][0]);
        acc[i][1] = fmaf(av[i], bv.y, acc[i][1]);
        acc[i][2] = fmaf(av[i], bv.z, acc[i][2]);
        acc[i][3] = fmaf(av[i], bv.w, acc[i][3]);
      }
    }
    __syncthreads();
  }
  float cs[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t gn = n0 + tn * 4 + j;
    cs[j] = (colscale && gn < N ? colscale[gn] : 1.f) * alpha;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t gm = m0 + tm * 8 + i;
    if (gm >= M) continue;
    const int64_t row = rowmap ? (int64_t)rowmap[gm] : gm;
    if (row < 0) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + tn * 4 + j;
      if (gn >= N) continue;
      const float v = acc[i][j] * cs[j];
      float* dst = C + row * ldc + gn;
      *dst = accumulate ? *dst + v : v;
    }
  }
}

int gemm_ts(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda, int asum,
            int64_t astride, const float* B, int64_t ldb, const float* colscale, float* C,
            int64_t ldc, const int32_t* rowmap, int accumulate, cudaStream_t s) {
  const int async_a = asum == 1 && K % 4 == 0 && lda % 4 == 0 &&
                      (reinterpret_cast<uintptr_t>(A) & 15) == 0;
  const int async_b = N % 4 == 0 && ldb % 4 == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0;
  const int64_t max_rows = (int64_t)65535 * SBM;
  for (int64_t r0 = 0; r0 < M; r0 += max_rows) {
    const int64_t mm = M - r0 < max_rows ? M - r0 : max_rows;
    dim3 grid(ceil_div(N, SBN), ceil_div(mm, SBM));
    gemm_ts_kernel<<<grid, 256, 0, s>>>(mm, N, K, alpha, A + r0 * lda, lda, asum, astride, B, ldb,
                                       colscale, rowmap ? C : C + r0 * ldc, ldc,
                                       rowmap ? rowmap + r0 : nullptr, accumulate, async_a,
                                       async_b);
  }
  return launch_status();
}

// ---------------------------------------------------------------------------
// float64 GEMM on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64), same
// contract as gemm_kernel (split-sum A loader, colscale, alpha, accumulate,
// row scatter).  CTA tile 128 x 64, 8 warps as 4 (M) x 2 (N), warp tile
// 32 x 32 = 4 x 4 m8n8 fragments; 16-deep K stages, double-buffered: cp.async
// straight to shared memory when A (asum == 1) and B rows are 16-byte
// aligned, a register-staged loader otherwise.  Padded shared strides keep
// the fragment loads conflict-free.
constexpr int DBM = 128, DBN = 64, DBK = 16;
constexpr int DAS = DBK + 4;    // A tile row stride (doubles)
constexpr int DBS = DBN + 4;    // B tile row stride (doubles): = 4 mod 16, the 16 lanes of a half-warp (rows lane & 3, columns lane >> 2) hit 16 distinct bank pairs

__device__ __forceinline__ void dmma_884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) gemm_dmma_kernel(
    int64_t M, int64_t N, int64_t K, double alpha, const double* __restrict__ A, int64_t lda,
    int asum, int64_t astride, const double* __restrict__ B, int64_t ldb,
    const double* __restrict__ colscale, double* __restrict__ C, int64_t ldc,
    const int32_t* __restrict__ rowmap, int accumulate, int async_a, int async_b) {
  extern __shared__ __align__(16) double dg_smem[];
  double (*As)[DBM * DAS] = reinterpret_cast<double (*)[DBM * DAS]>(dg_smem);
  double (*Bs)[DBK * DBS] = reinterpret_cast<double (*)[DBK * DBS]>(dg_smem + 2 * DBM * DAS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;
  const int64_t m0 = (int64_t)blockIdx.y * DBM, n0 = (int64_t)blockIdx.x * DBN;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto stage = [&](int64_t k0, int buf) {
    // A: 128 rows x 16 doubles = 8 chunks of 2 per row; thread -> (row, chunk)
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int e = tid + it * 256;
      const int r = e >> 3, c = (e & 7) * 2;
      const int64_t gm = m0 + r, gk = k0 + c;
      double* dst = &As[buf][r * DAS + c];
      if (async_a) {
        const bool ok = gm < M && gk < K;         // K even: the pair is in or out together
        cp_async16(dst, ok ? A + gm * lda + gk : A, ok);
      } else {
        double v0 = 0.0, v1 = 0.0;
        if (gm < M) {
          const double* p = A + gm * lda;
          for (int q = 0; q < asum; ++q) {
            if (gk < K) v0 += p[q * astride + gk];
            if (gk + 1 < K) v1 += p[q * astride + gk + 1];
          }
        }
        dst[0] = v0;
        dst[1] = v1;
      }
    }
    // B: 16 rows x 64 doubles = 32 chunks of 2 per row
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int e = tid + it * 256;
      const int r = e >> 5, c = (e & 31) * 2;
      const int64_t gk = k0 + r, gn = n0 + c;
      double* dst = &Bs[buf][r * DBS + c];
      if (async_b) {
        const bool ok = gk < K && gn < N;         // N even
        cp_async16(dst, ok ? B + gk * ldb + gn : B, ok);
      } else {
        dst[0] = (gk < K && gn < N) ? B[gk * ldb + gn] : 0.0;
        dst[1] = (gk < K && gn + 1 < N) ? B[gk * ldb + gn + 1] : 0.0;
      }
    }
    cp_async_commit();
  };

  const int nk = (int)((K + DBK - 1) / DBK);
  stage(0, 0);
  const int arow = 32 * wm + (lane >> 2), acol = lane & 3;
  const int bcol = 32 * wn + (lane >> 2), brow = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) {
      stage((int64_t)(kt + 1) * DBK, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* a = &As[buf][arow * DAS + acol];
    const double* b = &Bs[buf][brow * DBS + bcol];
#pragma unroll
    for (int ks = 0; ks < DBK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = a[i * 8 * DAS + ks];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = b[ks * DBS + j * 8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_884(acc[i][j], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + 32 * wm + 8 * i + (lane >> 2);
    if (gm >= M) continue;
    const int64_t row = rowmap ? (int64_t)rowmap[gm] : gm;
    if (row < 0) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gn = n0 + 32 * wn + 8 * j + 2 * (lane & 3) + h;
        if (gn >= N) continue;
        double v = acc[i][j][h];
        if (colscale) v *= colscale[gn];
        v *= alpha;
        double* dst = C + row * ldc + gn;
        *dst = accumulate ? *dst + v : v;
      }
    }
  }
}

int gemm_dmma(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
              int asum, int64_t astride, const double* B, int64_t ldb, const double* colscale,
              double* C, int64_t ldc, const int32_t* rowmap, int accumulate, cudaStream_t s) {
  const int async_a = asum == 1 && K % 2 == 0 && lda % 2 == 0 &&
                      (reinterpret_cast<uintptr_t>(A) & 15) == 0;
  const int async_b = N % 2 == 0 && ldb % 2 == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0;
  constexpr size_t kSmem = sizeof(double) * (2 * DBM * DAS + 2 * DBK * DBS);
  set_max_smem((const void*)gemm_dmma_kernel, kSmem);
  const int64_t max_rows = (int64_t)65535 * DBM;
  for (int64_t r0 = 0; r0 < M; r0 += max_rows) {
    const int64_t mm = M - r0 < max_rows ? M - r0 : max_rows;
    dim3 grid(ceil_div(N, DBN), ceil_div(mm, DBM));
    gemm_dmma_kernel<<<grid, 256, kSmem, s>>>(mm, N, K, alpha, A + r0 * lda, lda, asum, astride, B, ldb,
                                          colscale, rowmap ? C : C + r0 * ldc, ldc,
                                          rowmap ? rowmap + r0 : nullptr, accumulate, async_a,
                                          async_b);
  }
  return launch_status();
}

template <typename T>
__global__ void stack_kernel(const T* __restrict__ mult, const int32_t* __restrict__ child,
                             int64_t n_par, int64_t nrhs, int64_t ne, T* __restrict__ out) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t width = 8 * ne;
  if (idx >= n_par * nrhs * width) return;
  int64_t row = idx / width, col = idx - row * width;
  int64_t p = row / nrhs, r = row - p * nrhs;
  int c = (int)(col / ne);
  int64_t e = col - (int64_t)c * ne;
  int32_t ch = child[p * 8 + c];
  out[idx] = ch >= 0 ? mult[((int64_t)ch * nrhs + r) * ne + e] : T(0);
}

template <typename T>
int stack(const T* mult, const int32_t* child, int64_t n_par, int64_t nrhs, int64_t ne, T* out,
          void* stream) {
  if (n_par < 0 || nrhs < 1 || ne < 1) return KIFMM_EARG;
  int64_t total = n_par * nrhs * 8 * ne;
  if (total == 0) return 0;
  stack_kernel<T><<<ceil_div(total, 256), 256, 0, (cudaStream_t)stream>>>(mult, child, n_par,
                                                                          nrhs, ne, out);
  return launch_status();
}

template <typename T>
__global__ void gather_charges_kernel(const double* __restrict__ qin,
                                      const int64_t* __restrict__ perm, int64_t n, int64_t nrhs,
                                      T* __restrict__ qt) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * nrhs) return;
  int64_t i = idx / nrhs, r = idx - i * nrhs;
  qt[idx] = (T)qin[perm[i] * nrhs + r];
}

// Charge intake in one pass: qt[i*nrhs + r] = (T) qin[perm[i]*nrhs + r] (caller
// order, float64 -> tree order, working type) and the packed source record
// src4[r*n + i] = (x_i, y_i, z_i, q).  Four points per thread, a block-stride
// apart: four independent gather chains in flight (the permuted read is
// latency-bound) with every access still coalesced across the warp.
template <typename T, typename V4>
__global__ void __launch_bounds__(256) gather_pack_kernel(
    const double* __restrict__ qin, const int64_t* __restrict__ perm, const T* __restrict__ sx,
    const T* __restrict__ sy, const T* __restrict__ sz, int64_t n, int64_t nrhs,
    T* __restrict__ qt, V4* __restrict__ src4) {
  const int64_t base = (int64_t)blockIdx.x * (4 * 256) + threadIdx.x;
  int64_t pi[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t i = base + u * 256;
    pi[u] = i < n ? perm[i] : 0;
  }
  for (int64_t r = 0; r < nrhs; ++r) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = base + u * 256 < n ? qin[pi[u] * nrhs + r] : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = base + u * 256;
      if (i < n) {
        const T qv = (T)v[u];
        qt[i * nrhs + r] = qv;
        src4[r * n + i] = V4{sx[i], sy[i], sz[i], qv};
      }
    }
  }
}

// Row gather/scatter of width-element rows (multipole halo pack/unpack).
template <typename T>
__global__ void rows_kernel(const T* __restrict__ src, const int32_t* __restrict__ rows,
                            int64_t n_rows, int64_t width, T* __restrict__ dst, int scatter) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_rows * width) return;
  const int64_t i = idx / width, e = idx - i * width;
  const int64_t g = rows[i];
  if (scatter == 2) {                      // scatter-add; rows < 0 are skipped
    if (g >= 0) dst[g * width + e] += src[idx];
  } else if (scatter) {
    dst[g * width + e] = src[idx];
  } else {
    dst[idx] = src[g * width + e];
  }
}

// dst[dst_rows[i]] = src[src_rows[i]] (halo unpack straight out of an
// all-gathered buffer: no intermediate copy)
template <typename T>
__global__ void move_rows_kernel(const T* __restrict__ src, const int32_t* __restrict__ src_rows,
                                 const int32_t* __restrict__ dst_rows, int64_t n_rows,
                                 int64_t width, T* __restrict__ dst) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_rows * width) return;
  const int64_t i = idx / width, e = idx - i * width;
  dst[(int64_t)dst_rows[i] * width + e] = src[(int64_t)src_rows[i] * width + e];
}

template <typename T>
int move_rows(const T* src, const int32_t* src_rows, const int32_t* dst_rows, int64_t n_rows,
              int64_t width, T* dst, void* stream) {
  if (n_rows < 0 || width < 1) return KIFMM_EARG;
  if (n_rows == 0) return 0;
  move_rows_kernel<T><<<ceil_div(n_rows * width, 256), 256, 0, (cudaStream_t)stream>>>(
      src, src_rows, dst_rows, n_rows, width, dst);
  return launch_status();
}

template <typename T>
int rows_op(const T* src, const int32_t* rows, int64_t n_rows, int64_t width, T* dst, int scatter,
            void* stream) {
  if (n_rows < 0 || width < 1) return KIFMM_EARG;
  if (n_rows == 0) return 0;
  rows_kernel<T><<<ceil_div(n_rows * width, 256), 256, 0, (cudaStream_t)stream>>>(
      src, rows, n_rows, width, dst, scatter);
  return launch_status();
}

}  // namespace

extern "C" {

int kifmm_gather_rows_f32(const float* src, const int32_t* rows, int64_t n_rows, int64_t width,
                          float* dst, void* s) {
  return rows_op<float>(src, rows, n_rows, width, dst, 0, s);
}
int kifmm_gather_rows_f64(const double* src, const int32_t* rows, int64_t n_rows, int64_t width,
                          double* dst, void* s) {
  return rows_op<double>(src, rows, n_rows, width, dst, 0, s);
}
int kifmm_scatter_rows_f32(const float* src, const int32_t* rows, int64_t n_rows, int64_t width,
                           float* dst, void* s) {
  return rows_op<float>(src, rows, n_rows, width, dst, 1, s);
}
int kifmm_scatter_rows_f64(const double* src, const int32_t* rows, int64_t n_rows, int64_t width,
                           double* dst, void* s) {
  return rows_op<double>(src, rows, n_rows, width, dst, 1, s);
}

int kifmm_move_rows_f32(const float* src, const int32_t* src_rows, const int32_t* dst_rows,
                        int64_t n_rows, int64_t width, float* dst, void* s) {
  return move_rows<float>(src, src_rows, dst_rows, n_rows, width, dst, s);
}
int kifmm_move_rows_f64(const double* src, const int32_t* src_rows, const int32_t* dst_rows,
                        int64_t n_rows, int64_t width, double* dst, void* s) {
  return move_rows<double>(src, src_rows, dst_rows, n_rows, width, dst, s);
}

int kifmm_scatter_add_rows_f32(const float* src, const int32_t* rows, int64_t n_rows,
                               int64_t width, float* dst, void* s) {
  return rows_op<float>(src, rows, n_rows, width, dst, 2, s);
}
int kifmm_scatter_add_rows_f64(const double* src, const int32_t* rows, int64_t n_rows,
                               int64_t width, double* dst, void* s) {
  return rows_op<double>(src, rows, n_rows, width, dst, 2, s);
}

int kifmm_gemm_f32(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda,
                   int asum, int64_t astride, const float* B, int64_t ldb, const float* colscale,
                   float* C, int64_t ldc, const int32_t* rowmap, int accumulate, void* s) {
  if (M < 0 || N < 0 || K < 0 || asum < 1) return KIFMM_EARG;
  if (M == 0 || N == 0) return 0;
  // tall shapes: the 128-row cp.async kernel, else the SIMT tiles
  if (M * ((N + SBN - 1) / SBN) >= 128 * 148)
    return gemm_ts(M, N, K, alpha, A, lda, asum, astride, B, ldb, colscale, C, ldc, rowmap,
                   accumulate, (cudaStream_t)s);
  return gemm<float>(M, N, K, alpha, A, lda, asum, astride, B, ldb, colscale, C, ldc, rowmap,
                     accumulate, s);
}
int kifmm_gemm_f64(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                   int asum, int64_t astride, const double* B, int64_t ldb,
                   const double* colscale, double* C, int64_t ldc, const int32_t* rowmap,
                   int accumulate, void* s) {
  // FP64 tensor cores for every tile-worthy shape
  if (M >= 256 && N >= 8 && K >= 4 && asum >= 1)
    return gemm_dmma(M, N, K, alpha, A, lda, asum, astride, B, ldb, colscale, C, ldc, rowmap,
                     accumulate, (cudaStream_t)s);
  return gemm<double>(M, N, K, alpha, A, lda, asum, astride, B, ldb, colscale, C, ldc, rowmap,
                      accumulate, s);
}
int kifmm_stack_children_f32(const float* mult, const int32_t* child, int64_t n_par, int64_t nrhs,
                             int64_t ne, float* out, void* s) {
  return stack<float>(mult, child, n_par, nrhs, ne, out, s);
}
int kifmm_stack_children_f64(const double* mult, const int32_t* child, int64_t n_par,
                             int64_t nrhs, int64_t ne, double* out, void* s) {
  return stack<double>(mult, child, n_par, nrhs, ne, out, s);
}
int kifmm_gather_pack_f32(const double* qin, const int64_t* perm, const float* sx, const float* sy,
                          const float* sz, int64_t n, int64_t nrhs, float* qt, float* src4,
                          void* s) {
  if (n < 0 || nrhs < 1) return KIFMM_EARG;
  if (n == 0) return 0;
  gather_pack_kernel<float, float4><<<ceil_div(n, 4 * 256), 256, 0, (cudaStream_t)s>>>(
      qin, perm, sx, sy, sz, n, nrhs, qt, reinterpret_cast<float4*>(src4));
  return launch_status();
}
int kifmm_gather_pack_f64(const double* qin, const int64_t* perm, const double* sx,
                          const double* sy, const double* sz, int64_t n, int64_t nrhs, double* qt,
                          double* src4, void* s) {
  if (n < 0 || nrhs < 1) return KIFMM_EARG;
  if (n == 0) return 0;
  gather_pack_kernel<double, double4><<<ceil_div(n, 4 * 256), 256, 0, (cudaStream_t)s>>>(
      qin, perm, sx, sy, sz, n, nrhs, qt, reinterpret_cast<double4*>(src4));
  return launch_status();
}
int kifmm_gather_charges_f32(const double* qin, const int64_t* perm, int64_t n, int64_t nrhs,
                             float* qt, void* s) {
  if (n < 0 || nrhs < 1) return KIFMM_EARG;
  if (n == 0) return 0;
  gather_charges_kernel<float><<<ceil_div(n * nrhs, 256), 256, 0, (cudaStream_t)s>>>(qin, perm, n,
                                                                                   nrhs, qt);
  return launch_status();
}
int kifmm_gather_charges_f64(const double* qin, const int64_t* perm, int64_t n, int64_t nrhs,
                             double* qt, void* s) {
  if (n < 0 || nrhs < 1) return KIFMM_EARG;
  if (n == 0) return 0;
  gather_charges_kernel<double><<<ceil_div(n * nrhs, 256), 256, 0, (cudaStream_t)s>>>(
      qin, perm, n, nrhs, qt);
  return launch_status();
}

}  // extern "C"
