// Fused row chain for tall inputs and narrow operators (float32, every
// operator dimension <= 64):
//
//   Y0 = X . B0 (x cs0, x al0);  Y1 = Y0 . B1 (x cs1, x al1);  Y2 = Y1 . B2 ...
//
// with an optional global output after EVERY stage (plain, accumulated, or
// through a destination row map).  One CTA takes 128 input rows; the row
// tile and its intermediates stay in shared memory, each operator is staged
// once per CTA, and a thread owns an 8 x 4 block of the stage output
// (LDS.128 for both operands: 12 shared loads per 128 FMAs).
//
// The evaluate uses it where a chain of small GEMMs over all boxes of the
// leaf level sat on the critical path in front of the finest M2L sweep:
//   P2M solve + M2L projection   phi . U_up (x inv) . V_up^T (x side) -> multipoles,
//                                . S -> q~ rows of the dense sub-lattice array
//   (reference expansion.py:78-82 through engine.py:298-318, then
//   m2l_blas.py:284-288); three launches (~70 us at 32768 leaves, each
//   latency-bound) become one.
// The chain kernel of chain.cu covers the same algebra for small row counts
// and wide operators; this one is sized for M >= ~16k rows.
#include "common.cuh"

using namespace kifmm;

namespace {

constexpr int BM = 128;        // input rows per CTA
constexpr int XS = 68;         // row stride of the staged tiles (floats): 16-byte aligned rows
constexpr int BW = 64;         // operator width limit and row stride of the staged operator
constexpr int NTH = 256;

struct RowChainArgs {
  int64_t M;
  const float* A;
  int64_t lda;
  int asum;                    // X[m][k] = sum_{s < asum} A[m*lda + s*astride + k]
  int64_t astride;
  int nstage;
  const float* B[3];           // (K, N) row-major, ld = N
  int K[3], N[3];
  const float* cs[3];          // optional column scale (N)
  float al[3];
  float* C[3];                 // optional output of the stage
  int64_t ldc[3];
  const int32_t* rowmap[3];    // optional destination row of input row g (< 0: skipped)
  int accumulate[3];
};

__global__ void __launch_bounds__(NTH, 2) rowchain_kernel(const RowChainArgs a) {
  extern __shared__ __align__(16) float smem[];
  float* X0 = smem;
  float* X1 = X0 + BM * XS;
  float* Bs = X1 + BM * XS;                          // [64][BW]
  const int tid = threadIdx.x;
  const int64_t row0 = (int64_t)blockIdx.x * BM;
  const int rows_in = (int)min64(BM, a.M - row0);

  // ---- X tile (split-sum at the load), columns padded with zeros to a multiple of 4
  {
    const int K0 = a.K[0], K4 = (K0 + 3) & ~3;
    const bool vec = (K0 % 4 == 0) && (a.lda % 4 == 0) && (a.astride % 4 == 0) &&
                     ((reinterpret_cast<uintptr_t>(a.A) & 15) == 0);
    if (vec) {
      const int cpr = K0 / 4;
      for (int e = tid; e < BM * cpr; e += NTH) {
        const int m = e / cpr, c = e - m * cpr;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (m < rows_in) {
          const float* p = a.A + (row0 + m) * a.lda + 4 * c;
          v = __ldg(reinterpret_cast<const float4*>(p));
          for (int s = 1; s < a.asum; ++s) {
            const float4 w = __ldg(reinterpret_cast<const float4*>(p + s * a.astride));
            v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
          }
        }
        *reinterpret_cast<float4*>(X0 + m * XS + 4 * c) = v;
      }
    } else {
      for (int e = tid; e < BM * K4; e += NTH) {
        const int m = e / K4, k = e - m * K4;
        float v = 0.f;
        if (m < rows_in && k < K0) {
          const float* p = a.A + (row0 + m) * a.lda + k;
          v = __ldg(p);
          for (int s = 1; s < a.asum; ++s) v += __ldg(p + s * a.astride);
        }
        X0[m * XS + k] = v;
      }
    }
  }

  const int ty = tid >> 4, tx = tid & 15;            // rows ty*8 .. +7, columns tx*4 .. +3
  float* in = X0;
  float* out = X1;
  for (int s = 0; s < a.nstage; ++s) {
    const int K = a.K[s], N = a.N[s], K4 = (K + 3) & ~3;
    // ---- operator: rows K..K4 and columns N..BW zero
    {
      const float* B = a.B[s];
      for (int e = tid; e < K4 * BW; e += NTH) {
        const int k = e / BW, n = e - k * BW;
        Bs[e] = (k < K && n < N) ? __ldg(B + (int64_t)k * N + n) : 0.f;
      }
    }
    __syncthreads();
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[i][c] = 0.f;
    if (tx * 4 < N) {
#pragma unroll 2
      for (int k = 0; k < K4; k += 4) {
        const float4 b0 = *reinterpret_cast<const float4*>(Bs + (k + 0) * BW + tx * 4);
        const float4 b1 = *reinterpret_cast<const float4*>(Bs + (k + 1) * BW + tx * 4);
        const float4 b2 = *reinterpret_cast<const float4*>(Bs + (k + 2) * BW + tx * 4);
        const float4 b3 = *reinterpret_cast<const float4*>(Bs + (k + 3) * BW + tx * 4);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 x = *reinterpret_cast<const float4*>(in + (ty * 8 + i) * XS + k);
          acc[i][0] = fmaf(x.w, b3.x, fmaf(x.z, b2.x, fmaf(x.y, b1.x, fmaf(x.x, b0.x, acc[i][0]))));
          acc[i][1] = fmaf(x.w, b3.y, fmaf(x.z, b2.y, fmaf(x.y, b1.y, fmaf(x.x, b0.y, acc[i][1]))));
          acc[i][2] = fmaf(x.w, b3.z, fmaf(x.z, b2.z, fmaf(x.y, b1.z, fmaf(x.x, b0.z, acc[i][2]))));
          acc[i][3] = fmaf(x.w, b3.w, fmaf(x.z, b2.w, fmaf(x.y, b1.w, fmaf(x.x, b0.w, acc[i][3]))));
        }
      }
    }
    // ---- scale, hand over to the next stage, optional global output
    float sc[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int n = tx * 4 + c;
      sc[c] = a.al[s] * ((a.cs[s] && n < N) ? __ldg(a.cs[s] + n) : 1.f);
    }
    float* C = a.C[s];
    const bool vecout = C && (N % 4 == 0) && (a.ldc[s] % 4 == 0) &&
                        ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = ty * 8 + i;
      const float4 y = make_float4(acc[i][0] * sc[0], acc[i][1] * sc[1], acc[i][2] * sc[2],
                                   acc[i][3] * sc[3]);
      *reinterpret_cast<float4*>(out + m * XS + tx * 4) = y;     // columns >= N are zeros
      if (C && m < rows_in && tx * 4 < N) {
        const int64_t g = row0 + m;
        const int64_t dst = a.rowmap[s] ? (int64_t)a.rowmap[s][g] : g;
        if (dst >= 0) {
          float* o = C + dst * a.ldc[s] + tx * 4;
          if (vecout) {
            float4 v = y;
            if (a.accumulate[s]) {
              const float4 w = *reinterpret_cast<const float4*>(o);
              v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
            }
            *reinterpret_cast<float4*>(o) = v;
          } else {
            const float yy[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (tx * 4 + c < N) o[c] = a.accumulate[s] ? o[c] + yy[c] : yy[c];
          }
        }
      }
    }
    __syncthreads();
    float* t = in;
    in = out;
    out = t;
  }
}

}  // namespace

extern "C" {

// Fused row chain (see the header of this file).  Stage s: operator B_s
// (K_s x N_s, row-major), optional column scale cs_s (N_s), scalar al_s,
// optional output C_s (ldc_s, optional int32 row map over the M input rows,
// accumulate flag).  K_0 <= 64, N_s <= 64, K_{s+1} = N_s.
int kifmm_rowchain_f32(int64_t M, const float* A, int64_t lda, int64_t asum, int64_t astride,
                       int64_t nstage, const float* B0, const float* B1, const float* B2,
                       int64_t K0, int64_t N0, int64_t N1, int64_t N2, const float* cs0,
                       const float* cs1, const float* cs2, float al0, float al1, float al2,
                       float* C0, float* C1, float* C2, int64_t ldc0, int64_t ldc1, int64_t ldc2,
                       const int32_t* map0, const int32_t* map1, const int32_t* map2, int64_t acc0,
                       int64_t acc1, int64_t acc2, void* stream) {
  if (M < 0 || nstage < 1 || nstage > 3 || asum < 1 || !A) return KIFMM_EARG;
  const int64_t N[3] = {N0, N1, N2};
  const int64_t K[3] = {K0, N0, N1};
  const float* B[3] = {B0, B1, B2};
  for (int s = 0; s < nstage; ++s)
    if (K[s] < 1 || K[s] > BW || N[s] < 1 || N[s] > BW || !B[s]) return KIFMM_EARG;
  if (M == 0) return 0;
  RowChainArgs a;
  a.M = M;
  a.A = A;
  a.lda = lda;
  a.asum = (int)asum;
  a.astride = astride;
  a.nstage = (int)nstage;
  const float* cs[3] = {cs0, cs1, cs2};
  const float al[3] = {al0, al1, al2};
  float* C[3] = {C0, C1, C2};
  const int64_t ldc[3] = {ldc0, ldc1, ldc2};
  const int32_t* mp[3] = {map0, map1, map2};
  const int64_t ac[3] = {acc0, acc1, acc2};
  for (int s = 0; s < 3; ++s) {
    a.B[s] = B[s];
    a.K[s] = (int)K[s];
    a.N[s] = (int)N[s];
    a.cs[s] = cs[s];
    a.al[s] = al[s];
    a.C[s] = s < nstage ? C[s] : nullptr;
    a.ldc[s] = ldc[s];
    a.rowmap[s] = mp[s];
    a.accumulate[s] = (int)ac[s];
  }
  const size_t smem = sizeof(float) * (2 * BM * XS + 64 * BW);
  set_max_smem((const void*)rowchain_kernel, smem);
  rowchain_kernel<<<ceil_div(M, BM), NTH, smem, (cudaStream_t)stream>>>(a);
  return launch_status();
}

}  // extern "C"
