// Fused chains of small dense operators applied to a tile of rows:
//
//   Y0 = X . B0 (x cs0, x al0) ;  Y1 = Y0' . B1 (x cs1, x al1) ;  Y2 = Y1' . B2 ...
//
// where Ys' is Ys re-read as rows of width K(s+1) (K(s+1) divides N(s): the
// L2L product (parent, 8 children x n_check) becomes 8 child rows of n_check).
// Intermediates live in shared memory; only X is read and the last stage is
// written (optionally accumulated, optionally through a destination row map).
//
// This covers every operator chain of the evaluate around the hot path:
//   P2M solve       phi . U_up (x inv) . V_up^T (x side)       (expansion.py:78-82)
//   M2M             stack(children) . M2M^T . U_up (x inv) . V_up^T   (engine.py:321-334)
//   M2L epilogue    sum_splits(acc) . U^T (x 1/side) . U_dn (x inv) . V_dn^T (x side)
//                   (m2l_blas.py:322 + engine.py:355)
//   L2L             local . L2L^T -> per child . U_dn (x inv) . V_dn^T (x 0.5) -> scatter
//                   (engine.py:358-374)
// and keeps the reference's factored order (kernel product, then the solve).
#include "common.cuh"

using namespace kifmm;

namespace {

constexpr int NT = 256;

struct ChainArgs {
  int64_t M;                 // input rows
  int bm;                    // input rows per CTA
  int nstage;
  int64_t lda;
  int asum;
  int64_t astride;
  const int32_t* a_child;    // optional: row (p, r) = concat over children c of src row a_child[p*8+c]*R + r
  int64_t child_rows_w;      // width of one child row when a_child is set
  int64_t a_nrhs;            // R for the child-stack mode
  int64_t per_row;           // widest per-input-row footprint over the stages
  int64_t K[3], N[3];
  const void* B[3];
  const void* cs[3];
  double al[3];
  int64_t ldc;
  const int32_t* c_rowmap;
  int accumulate;
};

constexpr int RC = 4;          // consecutive output columns per work item
constexpr int RR = 4;          // rows per work item
constexpr int MAXIPT = 4;      // work items per thread
constexpr int BS_BYTES = 48 * 1024;   // operator K-chunk staged in shared memory

template <typename T>
__global__ void __launch_bounds__(NT) chain_kernel(const T* __restrict__ A, ChainArgs a,
                                                   T* __restrict__ C) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int64_t row0 = (int64_t)blockIdx.x * a.bm;
  const int rows_in = (int)min64(a.bm, a.M - row0);
  T* buf0 = reinterpret_cast<T*>(smem_raw);
  T* buf1 = buf0 + (int64_t)a.bm * a.per_row;
  T* Bs = buf1 + (int64_t)a.bm * a.per_row;

  // load the X tile: U independent loads in flight per thread (the split-sum
  // and child-stack reads are latency-bound when the tile is small).
  const int64_t K0 = a.K[0];
  auto load_x = [&](int64_t e) -> T {
    const int m = (int)(e / K0);
    const int64_t k = e - (int64_t)m * K0;
    if (m >= rows_in) return T(0);
    const int64_t g = row0 + m;
    if (a.a_child) {
      const int c = (int)(k / a.child_rows_w);
      const int64_t p = g / a.a_nrhs, r = g - p * a.a_nrhs;
      const int32_t ch = a.a_child[p * 8 + c];
      return ch >= 0 ? __ldg(&A[((int64_t)ch * a.a_nrhs + r) * a.lda + (k - c * a.child_rows_w)])
                     : T(0);
    }
    const T* p = A + g * a.lda + k;
    T v = __ldg(p);
    int s = 1;
    for (; s + 4 <= a.asum; s += 4) {
      const T v1 = __ldg(p + s * a.astride), v2 = __ldg(p + (s + 1) * a.astride);
      const T v3 = __ldg(p + (s + 2) * a.astride), v4 = __ldg(p + (s + 3) * a.astride);
      v += v1; v += v2; v += v3; v += v4;
    }
    for (; s < a.asum; ++s) v += __ldg(p + s * a.astride);
    return v;
  };
  {
    constexpr int U = 8;
    const int64_t total = (int64_t)a.bm * K0;
    for (int64_t e0 = tid; e0 < total; e0 += (int64_t)NT * U) {
      T v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = e0 + (int64_t)u * NT;
        v[u] = e < total ? load_x(e) : T(0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = e0 + (int64_t)u * NT;
        if (e < total) buf0[e] = v[u];
      }
    }
  }

  T* in = buf0;
  T* outb = buf1;
  int64_t nrows = a.bm;            // rows of the current stage input
  int64_t expand = 1;              // output rows per input row of the chain
  for (int s = 0; s < a.nstage; ++s) {
    const int64_t K = a.K[s], N = a.N[s];
    const T* B = reinterpret_cast<const T*>(a.B[s]);
    const T* cs = reinterpret_cast<const T*>(a.cs[s]);
    const T al = (T)a.al[s];
    const bool last = s + 1 == a.nstage;
    const int64_t live_rows = (int64_t)rows_in * expand;
    const int64_t ncg = (N + RC - 1) / RC;
    const int64_t nrg = (nrows + RR - 1) / RR;
    const int64_t items = nrg * ncg;
    // Small tiles: split K over `ks` thread groups (reduced in shared memory
    // below) so the serial K loop per thread shrinks by ks.
    int ks = 1;
    while (ks < 8 && items * ks * 2 <= NT &&
           (int64_t)ks * 2 * nrows * N * (int64_t)sizeof(T) <= BS_BYTES)
      ks *= 2;
    const int64_t witems = items * ks;
    const int64_t kch = (BS_BYTES / (int64_t)sizeof(T)) / N;   // operator rows per chunk
    const bool vec = (N % RC == 0) && sizeof(T) == 4;
    T acc[MAXIPT][RR][RC];
#pragma unroll
    for (int i = 0; i < MAXIPT; ++i)
#pragma unroll
      for (int r = 0; r < RR; ++r)
#pragma unroll
        for (int j = 0; j < RC; ++j) acc[i][r][j] = T(0);
    for (int64_t k0 = 0; k0 < K; k0 += kch) {
      const int64_t kc = min64(kch, K - k0);
      __syncthreads();                                 // previous chunk consumed / X ready
      // operator chunk: contiguous kc*N elements, all copies in flight at once
      {
        const T* src = B + k0 * N;
        const int64_t bytes = kc * N * (int64_t)sizeof(T);
        if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(Bs)) & 15) == 0 &&
            (bytes & 15) == 0) {
          for (int64_t e = tid; e < bytes / 16; e += NT)
            cp_async16(reinterpret_cast<char*>(Bs) + 16 * e,
                       reinterpret_cast<const char*>(src) + 16 * e, true);
        } else {
          for (int64_t e = tid; e < kc * N; e += NT) {
            unsigned sa = (unsigned)__cvta_generic_to_shared(Bs + e);
            if constexpr (sizeof(T) == 8)
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src + e));
            else
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(src + e));
          }
        }
        cp_async_commit();
        cp_async_wait<0>();
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < MAXIPT; ++i) {
        const int64_t wit = tid + (int64_t)i * NT;
        if (wit < witems) {
          const int64_t it = wit % items;
          const int ksl = (int)(wit / items);
          const int64_t rg = it / ncg, n0 = (it - rg * ncg) * RC;
          const int64_t m0 = rg * RR;
          const T* x[RR];
#pragma unroll
          for (int r = 0; r < RR; ++r)
            x[r] = in + (m0 + r < nrows ? m0 + r : m0) * K + k0;
          const T* bp = Bs + n0;
#pragma unroll 4
          for (int k = ksl; k < (int)kc; k += ks) {
            T bv[RC];
            if (vec) {
              const float4 t4 = *reinterpret_cast<const float4*>(bp + k * N);
              bv[0] = t4.x; bv[1] = t4.y; bv[2] = t4.z; bv[3] = t4.w;
            } else {
#pragma unroll
              for (int j = 0; j < RC; ++j) bv[j] = n0 + j < N ? bp[k * N + j] : T(0);
            }
#pragma unroll
            for (int r = 0; r < RR; ++r) {
              const T xv = x[r][k];
#pragma unroll
              for (int j = 0; j < RC; ++j) acc[i][r][j] += xv * bv[j];
            }
          }
        }
      }
    }
    // epilogue of the stage
    auto apply = [&](int64_t m, int64_t n, T v) {
      if (cs) v *= __ldg(&cs[n]);
      v *= al;
      if (!last) {
        outb[m * N + n] = v;
      } else {
        const int64_t gr = row0 * expand + m;
        const int64_t dst = a.c_rowmap ? (int64_t)a.c_rowmap[gr] : gr;
        if (dst >= 0) {
          T* o = C + dst * a.ldc + n;
          *o = a.accumulate ? *o + v : v;
        }
      }
    };
    if (ks == 1) {
#pragma unroll
      for (int i = 0; i < MAXIPT; ++i) {
        const int64_t it = tid + (int64_t)i * NT;
        if (it >= items) continue;
        const int64_t rg = it / ncg, n0 = (it - rg * ncg) * RC;
#pragma unroll
        for (int r = 0; r < RR; ++r) {
          const int64_t m = rg * RR + r;
          if (m >= nrows || (last && m >= live_rows)) continue;
#pragma unroll
          for (int j = 0; j < RC; ++j)
            if (n0 + j < N) apply(m, n0 + j, acc[i][r][j]);
        }
      }
    } else {
      // split-K partials -> Bs (free once every thread is past the K loop)
      T* red = Bs;
      __syncthreads();
#pragma unroll
      for (int i = 0; i < MAXIPT; ++i) {
        const int64_t wit = tid + (int64_t)i * NT;
        if (wit >= witems) continue;
        const int64_t it = wit % items;
        const int ksl = (int)(wit / items);
        const int64_t rg = it / ncg, n0 = (it - rg * ncg) * RC;
#pragma unroll
        for (int r = 0; r < RR; ++r) {
          const int64_t m = rg * RR + r;
          if (m >= nrows) continue;
#pragma unroll
          for (int j = 0; j < RC; ++j)
            if (n0 + j < N) red[((int64_t)ksl * nrows + m) * N + n0 + j] = acc[i][r][j];
        }
      }
      __syncthreads();
      for (int64_t e = tid; e < nrows * N; e += NT) {
        const int64_t m = e / N, n = e - m * N;
        if (last && m >= live_rows) continue;
        T v = red[e];
        for (int q = 1; q < ks; ++q) v += red[(int64_t)q * nrows * N + e];
        apply(m, n, v);
      }
    }
    if (!last) {
      const int64_t total = nrows * N;
      nrows = total / a.K[s + 1];
      expand = nrows / a.bm;
      T* t = in;
      in = outb;
      outb = t;
    }
  }
}

template <typename T>
int chain(int64_t M, const T* A, int64_t lda, int asum, int64_t astride, const int32_t* a_child,
          int64_t child_w, int64_t a_nrhs, int nstage, const T* B0, const T* B1, const T* B2, int64_t K0,
          int64_t N0, int64_t K1, int64_t N1, int64_t K2, int64_t N2, const T* cs0, const T* cs1,
          const T* cs2, double al0, double al1, double al2, T* C, int64_t ldc,
          const int32_t* c_rowmap, int accumulate, void* stream) {
  if (M < 0 || nstage < 1 || nstage > 3 || asum < 1 || K0 < 1 || N0 < 1) return KIFMM_EARG;
  if (M == 0) return 0;
  ChainArgs a{};
  a.M = M;
  a.nstage = nstage;
  a.lda = lda;
  a.asum = asum;
  a.astride = astride;
  a.a_child = a_child;
  a.child_rows_w = child_w;
  a.a_nrhs = a_nrhs < 1 ? 1 : a_nrhs;
  a.K[0] = K0; a.N[0] = N0; a.K[1] = K1; a.N[1] = N1; a.K[2] = K2; a.N[2] = N2;
  a.B[0] = B0; a.B[1] = B1; a.B[2] = B2;
  a.cs[0] = cs0; a.cs[1] = cs1; a.cs[2] = cs2;
  a.al[0] = al0; a.al[1] = al1; a.al[2] = al2;
  a.ldc = ldc;
  a.c_rowmap = c_rowmap;
  a.accumulate = accumulate;
  // widest per-input-row footprint over the stages
  int64_t per_row = K0, width = 1;   // width = rows per input row at the current stage
  for (int s = 0; s < nstage; ++s) {
    if (a.K[s] < 1 || a.N[s] < 1) return KIFMM_EARG;
    const int64_t w = width * a.N[s];
    per_row = per_row > w ? per_row : w;
    if (s + 1 < nstage) {
      if (w % a.K[s + 1]) return KIFMM_EARG;
      width = w / a.K[s + 1];
    }
  }
  a.per_row = per_row;
  // rows per CTA: <= MAXIPT*NT work items per stage, smem for the ping-pong
  // tiles plus the operator chunk, and about one wave when rows are few
  auto fits = [&](int bm_) {
    int64_t rows_s = bm_;
    for (int s = 0; s < nstage; ++s) {
      if (((rows_s + RR - 1) / RR) * ((a.N[s] + RC - 1) / RC) > (int64_t)MAXIPT * NT)
        return false;
      if (s + 1 < nstage) rows_s = rows_s * a.N[s] / a.K[s + 1];
    }
    return 2 * (size_t)bm_ * per_row * sizeof(T) + BS_BYTES <= 200 * 1024;
  };
  int bm = 128;
  while (bm > 1 && !fits(bm)) bm /= 2;
  while (bm > 8 && (M + bm - 1) / bm < 148) bm /= 2;
  if (!fits(bm)) return KIFMM_EARG;
  for (int s = 0; s < nstage; ++s)
    if ((int64_t)(BS_BYTES / sizeof(T)) / a.N[s] < 1) return KIFMM_EARG;
  a.bm = bm;
  const size_t smem = 2 * (size_t)bm * per_row * sizeof(T) + BS_BYTES;
  set_max_smem((const void*)chain_kernel<T>, smem);
  chain_kernel<T><<<ceil_div(M, bm), NT, smem, (cudaStream_t)stream>>>(A, a, C);
  return launch_status();
}

}  // namespace

extern "C" {

int kifmm_chain_f32(int64_t M, const float* A, int64_t lda, int asum, int64_t astride,
                    const int32_t* a_child, int64_t child_w, int64_t a_nrhs, int nstage,
                    const float* B0,
                    const float* B1, const float* B2, int64_t K0, int64_t N0, int64_t K1,
                    int64_t N1, int64_t K2, int64_t N2, const float* cs0, const float* cs1,
                    const float* cs2, double al0, double al1, double al2, float* C, int64_t ldc,
                    const int32_t* c_rowmap, int accumulate, void* s) {
  return chain<float>(M, A, lda, asum, astride, a_child, child_w, a_nrhs, nstage, B0, B1, B2, K0, N0, K1,
                      N1, K2, N2, cs0, cs1, cs2, al0, al1, al2, C, ldc, c_rowmap, accumulate, s);
}
int kifmm_chain_f64(int64_t M, const double* A, int64_t lda, int asum, int64_t astride,
                    const int32_t* a_child, int64_t child_w, int64_t a_nrhs, int nstage,
                    const double* B0,
                    const double* B1, const double* B2, int64_t K0, int64_t N0, int64_t K1,
                    int64_t N1, int64_t K2, int64_t N2, const double* cs0, const double* cs1,
                    const double* cs2, double al0, double al1, double al2, double* C, int64_t ldc,
                    const int32_t* c_rowmap, int accumulate, void* s) {
  return chain<double>(M, A, lda, asum, astride, a_child, child_w, a_nrhs, nstage, B0, B1, B2, K0, N0, K1,
                       N1, K2, N2, cs0, cs1, cs2, al0, al1, al2, C, ldc, c_rowmap, accumulate, s);
}

}  // extern "C"
