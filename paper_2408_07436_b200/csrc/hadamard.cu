// FFT-M2L Hadamard stage (replaces _hot.hadamard_m2l, _hot.pyx:141-178):
//   phat[f, c, tau, r] += sum_o sum_sigma khat[f, o, tau, sigma] * qhat[f, halo[c, o], sigma, r]
//
// For a fixed frequency f and halo offset o this is an 8x8 complex block
// applied to the gathered spectra of the target clusters' source clusters: a
// small GEMM whose right-hand side is a gather.  One CTA owns (f, a tile of
// 256 target clusters): khat[f] (26 x 64 complex) sits in shared memory; for
// each of the 26 offsets the tile's 256 source-cluster spectra (8 children
// each) are gathered into shared memory with cp.async, double-buffered across
// offsets; every thread keeps a 4-cluster x 2-tau complex accumulator in
// registers for the whole sweep (64 complex MACs per gathered offset), so
// the FP64/FP32 FMA pipe, not the loads, sets the pace.  phat is read and
// written once.
#include <cstdlib>

#include "common.cuh"

using namespace kifmm;

namespace {

template <typename T> struct cx;
template <> struct cx<float> { using v = float2; };
template <> struct cx<double> { using v = double2; };

constexpr int HT = 256;      // threads
constexpr int HC = 256;      // target clusters per CTA
constexpr int CPT = 4;       // clusters per thread

// Shared-memory slot of (cluster, sigma) in a gathered tile: the sigma index
// is rotated by the cluster group so the 8 clusters read by one shared-memory
// phase hit distinct banks.
__device__ __forceinline__ int qslot(int cl, int sg) { return cl * 8 + (sg ^ ((cl >> 2) & 7)); }

template <typename C>
__device__ __forceinline__ void cp_async_c(C* dst, const C* src, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? (int)sizeof(C) : 0;
  if constexpr (sizeof(C) == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(n));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(n));
}

template <typename T>
__global__ void __launch_bounds__(HT, 2) hadamard_kernel(const typename cx<T>::v* __restrict__ khat,
                                                      const typename cx<T>::v* __restrict__ qhat,
                                                      const int64_t* __restrict__ halo,
                                                      typename cx<T>::v* __restrict__ phat,
                                                      int64_t nsc, int64_t ntc, int64_t nrhs) {
  using C = typename cx<T>::v;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* ks = reinterpret_cast<C*>(smem_raw);              // [26][8 sigma][8 tau]
  C* qs = ks + 26 * 64;                                // [2][HC * 8]
  const int tid = threadIdx.x;
  const int64_t f = blockIdx.x;
  const int64_t c_begin = (int64_t)blockIdx.y * HC;
  const int64_t r = blockIdx.z;
  const int tp = tid >> 6;                             // tau pair: taus 2tp, 2tp+1
  const int cg = tid & 63;                             // cluster group: clusters 4cg .. 4cg+3

  const C* kf = khat + f * (26 * 64);
  for (int e = tid; e < 26 * 64; e += HT) {
    const int o = e >> 6, tau = (e >> 3) & 7, sig = e & 7;
    ks[(o * 8 + sig) * 8 + tau] = kf[e];
  }
  const C* qf = qhat + f * nsc * 8 * nrhs;

  // Halo indices of the clusters this thread gathers (elements tid + k*HT,
  // cluster (tid >> 3) + 32k), loaded one offset ahead of their gather so the
  // index latency hides behind a compute phase.
  constexpr int EPT = HC * 8 / HT;
  int64_t hidx[EPT];
  auto load_halo = [&](int o) {
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int64_t c = c_begin + (tid >> 3) + k * (HT >> 3);
      hidx[k] = c < ntc ? __ldg(&halo[c * 26 + o]) : -1;
    }
  };
  auto gather = [&](int buf) {
    C* dst = qs + buf * HC * 8;
    const int sg = tid & 7;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int cl = (tid >> 3) + k * (HT >> 3);
      const int64_t s = hidx[k];
      const C* src = qf + ((s < 0 ? 0 : s) * 8 + sg) * nrhs + r;
      cp_async_c(dst + qslot(cl, sg), src, s >= 0);
    }
    cp_async_commit();
  };

  T acc_re[CPT][2], acc_im[CPT][2];
#pragma unroll
  for (int i = 0; i < CPT; ++i)
#pragma unroll
    for (int t = 0; t < 2; ++t) acc_re[i][t] = acc_im[i][t] = T(0);

  load_halo(0);
  gather(0);
  load_halo(1);
  for (int o = 0; o < 26; ++o) {
    const int buf = o & 1;
    if (o + 1 < 26) {
      gather(buf ^ 1);
      if (o + 2 < 26) load_halo(o + 2);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const C* q = qs + buf * HC * 8;
    const C* kk = ks + o * 64 + 2 * tp;
#pragma unroll
    for (int sg = 0; sg < 8; ++sg) {
      const C k0 = kk[sg * 8], k1 = kk[sg * 8 + 1];
#pragma unroll
      for (int i = 0; i < CPT; ++i) {
        const C v = q[qslot(cg * CPT + i, sg)];
        acc_re[i][0] = fma(k0.x, v.x, acc_re[i][0]);
        acc_re[i][0] = fma(-k0.y, v.y, acc_re[i][0]);
        acc_im[i][0] = fma(k0.x, v.y, acc_im[i][0]);
        acc_im[i][0] = fma(k0.y, v.x, acc_im[i][0]);
        acc_re[i][1] = fma(k1.x, v.x, acc_re[i][1]);
        acc_re[i][1] = fma(-k1.y, v.y, acc_re[i][1]);
        acc_im[i][1] = fma(k1.x, v.y, acc_im[i][1]);
        acc_im[i][1] = fma(k1.y, v.x, acc_im[i][1]);
      }
    }
    __syncthreads();
  }
  C* pf = phat + f * ntc * 8 * nrhs;
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int64_t c = c_begin + cg * CPT + i;
    if (c >= ntc) continue;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      C* p = pf + (c * 8 + 2 * tp + t) * nrhs + r;
      C old = *p;
      old.x += acc_re[i][t];
      old.y += acc_im[i][t];
      *p = old;
    }
  }
}

template <typename T>
int hadamard(const T* khat, const T* qhat, const int64_t* halo, T* phat, int64_t nf, int64_t nsc,
             int64_t ntc, int64_t nrhs, void* stream) {
  using C = typename cx<T>::v;
  if (nf < 0 || nsc < 0 || ntc < 0 || nrhs < 1) return KIFMM_EARG;
  if (nf == 0 || ntc == 0) return 0;
  const size_t smem = (26 * 64 + 2 * HC * 8) * sizeof(C);
  set_max_smem((const void*)hadamard_kernel<T>, smem);
  dim3 grid((unsigned)nf, ceil_div(ntc, HC), (unsigned)nrhs);
  hadamard_kernel<T><<<grid, HT, smem, (cudaStream_t)stream>>>(
      reinterpret_cast<const C*>(khat), reinterpret_cast<const C*>(qhat), halo,
      reinterpret_cast<C*>(phat), nsc, ntc, nrhs);
  return launch_status();
}


// ---------------------------------------------------------------------------
// Tiled Hadamard.  The 26 x 256 gathers of the kernel above touch only the
// ~600 distinct source clusters around a tile of 256 target clusters (a
// 10 x 10 x 6 brick for a full tree), so a host plan (m2l_fft.py
// plan_hadamard_tiles) lists, per tile, those sources and each
// (offset, target) -> shared-memory slot.  A CTA owns one tile and a chunk
// of frequencies: per frequency it stages the tile's sources and khat[f]
// ONCE into shared memory (double-buffered against the previous frequency's
// compute) and every (o, target) block reads its spectra from there.
//
// Thread map: warp w, lane l -> tau pair tp = l & 3 and lane group g = l >> 2;
// slot-table column p = 32w + 4g + j (j < 4) holds a target of coordinate
// parity class g (the plan's column order), so at offset o all 4 sources of
// a lane have parity class c = g ^ parity(o), which the plan makes their
// slot's u % 8.  Spectra are stored rotated (slot u, sigma at u*8 + (sigma ^
// u%8)); with c shared by a lane's 4 targets one XOR per sigma addresses all
// four, the 8 lane groups of a warp read 8 different banks, and khat
// (staged [o][sigma][tau]) is read at the same sigma by the whole warp, the
// 4 tau pairs in distinct banks.  Absent sources point at zero rows UMAX + c.
constexpr int TT = 256;        // targets per tile
constexpr int UMAX = 600;      // source slots per tile; slots UMAX..UMAX+7 are zero rows
constexpr int QROWS = UMAX + 8;
constexpr int FCH = 8;         // frequencies per CTA

__device__ __forceinline__ void dmma_884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <typename C> __device__ __forceinline__ C lds_c(unsigned a);
template <> __device__ __forceinline__ double2 lds_c<double2>(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
template <> __device__ __forceinline__ float2 lds_c<float2>(unsigned a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}

template <typename T>
__global__ void __launch_bounds__(256, 1) hadamard_tiled_kernel(
    const typename cx<T>::v* __restrict__ khat, const typename cx<T>::v* __restrict__ qhat,
    const int64_t* __restrict__ tile_begin, const int64_t* __restrict__ src_off,
    const int64_t* __restrict__ src, const int16_t* __restrict__ slots,
    const int16_t* __restrict__ tcol, int64_t nf, int64_t nsc, int64_t ntc, int64_t nrhs,
    int accumulate, typename cx<T>::v* __restrict__ phat) {
  using C = typename cx<T>::v;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* ks = reinterpret_cast<C*>(smem_raw);                        // [2][26][8 sigma][8 tau]
  C* qs = ks + 2 * 26 * 64;                                      // [2][QROWS * 8]
  int16_t* sl = reinterpret_cast<int16_t*>(qs + 2 * QROWS * 8);  // [26][TT]
  int* ss = reinterpret_cast<int*>(sl + 26 * TT);                // [UMAX] source cluster per slot
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int64_t t = blockIdx.x;
  const int64_t f0 = (int64_t)blockIdx.y * FCH;
  const int64_t r = blockIdx.z;
  const int nfc = (int)min64(FCH, nf - f0);
  const int64_t cb = tile_begin[t];
  const int64_t so = src_off[t];
  const int ns = (int)(src_off[t + 1] - so);

  {
    const int4* s4 = reinterpret_cast<const int4*>(slots + t * 26 * TT);
    int4* d4 = reinterpret_cast<int4*>(sl);
    for (int e = tid; e < 26 * TT * 2 / 16; e += 256) d4[e] = __ldg(&s4[e]);
    for (int e = tid; e < ns; e += 256) ss[e] = (int)__ldg(&src[so + e]);
    for (int e = tid; e < 2 * 64; e += 256)
      qs[(e >> 6) * QROWS * 8 + UMAX * 8 + (e & 63)] = C{T(0), T(0)};
  }
  const int tp = l & 3, g = l >> 2;
  const int c0 = 32 * w + 4 * g;
  int tgt[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) tgt[j] = __ldg(&tcol[t * TT + c0 + j]);
  const bool active = __any_sync(0xffffffffu, (tgt[0] >= 0) | (tgt[1] >= 0) | (tgt[2] >= 0) |
                                                  (tgt[3] >= 0));
  __syncthreads();

  auto stage = [&](int64_t f, int b) {
    const C* kf = khat + f * (26 * 64);
    C* kd = ks + b * 26 * 64;
    for (int e = tid; e < 26 * 64; e += 256) {
      const int o = e >> 6, tau = (e >> 3) & 7, sg = e & 7;
      cp_async_c(kd + (o * 8 + sg) * 8 + tau, kf + e, true);
    }
    C* qd = qs + b * QROWS * 8;
    const C* qf = qhat + f * nsc * 8 * nrhs + r;
    for (int e = tid; e < ns * 8; e += 256) {
      const int u = e >> 3, sg = e & 7;
      const int sc = ss[u];
      if (sc >= 0) cp_async_c(qd + u * 8 + (sg ^ (u & 7)), qf + ((int64_t)sc * 8 + sg) * nrhs, true);
    }
    cp_async_commit();
  };

  stage(f0, 0);
  for (int i = 0; i < nfc; ++i) {
    const int b = i & 1;
    if (i + 1 < nfc) {
      stage(f0 + i + 1, b ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (active) {
      const unsigned q0 = (unsigned)__cvta_generic_to_shared(qs + b * QROWS * 8);
      const C* kb = ks + b * 26 * 64 + 2 * tp;
      // Split accumulators (re = sum kx vx - sum ky vy, ...): every
      // accumulator takes one FMA per sigma, 32 independent chains.
      T are[4][2], aim[4][2], bre[4][2], bim[4][2];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) are[j][h] = aim[j][h] = bre[j][h] = bim[j][h] = T(0);
#pragma unroll 2
      for (int o = 0; o < 26; ++o) {
        const short4 s4 = *reinterpret_cast<const short4*>(sl + o * TT + c0);
        // Byte addresses of the 4 spectra rows with the rotation folded in:
        // row u is 128/64-byte aligned, so u*8 + (sigma ^ c) = (row ^ c) ^ sigma.
        const int c = s4.x & 7;
        const unsigned qa[4] = {(q0 + (unsigned)s4.x * 8u * sizeof(C)) ^ (c * (unsigned)sizeof(C)),
                                (q0 + (unsigned)s4.y * 8u * sizeof(C)) ^ (c * (unsigned)sizeof(C)),
                                (q0 + (unsigned)s4.z * 8u * sizeof(C)) ^ (c * (unsigned)sizeof(C)),
                                (q0 + (unsigned)s4.w * 8u * sizeof(C)) ^ (c * (unsigned)sizeof(C))};
        const C* kp = kb + o * 64;
#pragma unroll
        for (int sg = 0; sg < 8; ++sg) {
          const C k0 = kp[sg * 8], k1 = kp[sg * 8 + 1];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const C v = lds_c<C>(qa[j] ^ (unsigned)(sg * sizeof(C)));
            are[j][0] = fma(k0.x, v.x, are[j][0]);
            bre[j][0] = fma(k0.y, v.y, bre[j][0]);
            aim[j][0] = fma(k0.x, v.y, aim[j][0]);
            bim[j][0] = fma(k0.y, v.x, bim[j][0]);
            are[j][1] = fma(k1.x, v.x, are[j][1]);
            bre[j][1] = fma(k1.y, v.y, bre[j][1]);
            aim[j][1] = fma(k1.x, v.y, aim[j][1]);
            bim[j][1] = fma(k1.y, v.x, bim[j][1]);
          }
        }
      }
      C* pf = phat + (f0 + i) * ntc * 8 * nrhs + r;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (tgt[j] < 0) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          C* p = pf + ((cb + tgt[j]) * 8 + 2 * tp + h) * nrhs;
          C v{are[j][h] - bre[j][h], aim[j][h] + bim[j][h]};
          if (accumulate) {
            const C old = *p;
            v.x += old.x;
            v.y += old.y;
          }
          *p = v;
        }
      }
    }
    __syncthreads();
  }
}

// float64 variant on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64).  Per
// (frequency, offset) the tile's block product is a real GEMM
//   [Yre Yim] (256 x 16) += [Xre Xim] (256 x 16) . [[Kr^T, Ki^T], [-Ki^T, Kr^T]]
// (k = 2 sigma + part, n = 2 tau + part).  An m8 fragment's 8 rows are the
// 8 siblings of an octet (one per parity class: the A loads of a warp hit 16
// distinct 16-byte units, see uslot); B fragments are read from the complex
// khat in shared memory with the sign of -Ki applied per lane.  Staging,
// plan and zero rows are those of hadamard_tiled_kernel.
__global__ void __launch_bounds__(256, 1) hadamard_tiled_dmma_kernel(
    const double2* __restrict__ khat, const double2* __restrict__ qhat,
    const int64_t* __restrict__ tile_begin, const int64_t* __restrict__ src_off,
    const int64_t* __restrict__ src, const int16_t* __restrict__ slots,
    const int16_t* __restrict__ tcol, int64_t nf, int64_t nsc, int64_t ntc, int64_t nrhs,
    int accumulate, double2* __restrict__ phat) {
  using C = double2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* ks = reinterpret_cast<C*>(smem_raw);                        // [2][26][8 sigma][8 tau]
  C* qs = ks + 2 * 26 * 64;                                      // [2][QROWS * 8]
  int16_t* sl = reinterpret_cast<int16_t*>(qs + 2 * QROWS * 8);  // [26][TT]
  int* ss = reinterpret_cast<int*>(sl + 26 * TT);                // [UMAX]
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int64_t t = blockIdx.x;
  const int64_t f0 = (int64_t)blockIdx.y * FCH;
  const int64_t r = blockIdx.z;
  const int nfc = (int)min64(FCH, nf - f0);
  const int64_t cb = tile_begin[t];
  const int64_t so = src_off[t];
  const int ns = (int)(src_off[t + 1] - so);

  {
    const int4* s4 = reinterpret_cast<const int4*>(slots + t * 26 * TT);
    int4* d4 = reinterpret_cast<int4*>(sl);
    for (int e = tid; e < 26 * TT * 2 / 16; e += 256) d4[e] = __ldg(&s4[e]);
    for (int e = tid; e < ns; e += 256) ss[e] = (int)__ldg(&src[so + e]);
    for (int e = tid; e < 2 * 64; e += 256)
      qs[(e >> 6) * QROWS * 8 + UMAX * 8 + (e & 63)] = C{0.0, 0.0};
  }
  const int g8 = l >> 2, kq = l & 3;
  const int c0 = 32 * w + 4 * g8;        // slot-table columns of this lane's 4 m-tile rows
  int tgt[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) tgt[i] = __ldg(&tcol[t * TT + c0 + i]);
  const bool active = __any_sync(0xffffffffu, (tgt[0] >= 0) | (tgt[1] >= 0) | (tgt[2] >= 0) |
                                                  (tgt[3] >= 0));
  // B fragment coordinates: k = 4 ks + kq -> (sigma = 2 ks + (kq >> 1), pk = kq & 1);
  // n = 8 jn + g8 -> (tau = 4 jn + (g8 >> 1), pn = g8 & 1)
  const int pk = kq & 1, pn = g8 & 1;
  const int comp = pk ^ pn;                              // 0: Re K, 1: Im K
  const unsigned long long neg = (pk && !pn) ? 0x8000000000000000ull : 0ull;
  __syncthreads();

  auto stage = [&](int64_t f, int b) {
    const C* kf = khat + f * (26 * 64);
    C* kd = ks + b * 26 * 64;
    for (int e = tid; e < 26 * 64; e += 256) {
      const int o = e >> 6, tau = (e >> 3) & 7, sg = e & 7;
      // tau ^ 2 in odd sigma rows: a B-fragment load touches rows sigma,
      // sigma + 1 (16 doubles apart: the same banks) at columns tau, tau + 1 -
      // the swizzle moves the odd row's pair to the other bank group
      cp_async_c(kd + (o * 8 + sg) * 8 + (tau ^ ((sg & 1) << 1)), kf + e, true);
    }
    C* qd = qs + b * QROWS * 8;
    const C* qf = qhat + f * nsc * 8 * nrhs + r;
    for (int e = tid; e < ns * 8; e += 256) {
      const int u = e >> 3, sg = e & 7;
      const int sc = ss[u];
      if (sc >= 0) cp_async_c(qd + u * 8 + (sg ^ (u & 7)), qf + ((int64_t)sc * 8 + sg) * nrhs, true);
    }
    cp_async_commit();
  };

  stage(f0, 0);
  for (int i = 0; i < nfc; ++i) {
    const int b = i & 1;
    if (i + 1 < nfc) {
      stage(f0 + i + 1, b ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (active) {
      const double* q = reinterpret_cast<const double*>(qs + b * QROWS * 8);
      const double* kb = reinterpret_cast<const double*>(ks + b * 26 * 64);
      double acc[4][2][2];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int jn = 0; jn < 2; ++jn) acc[m][jn][0] = acc[m][jn][1] = 0.0;
#pragma unroll 2
      for (int o = 0; o < 26; ++o) {
        const short4 s4 = *reinterpret_cast<const short4*>(sl + o * TT + c0);
        const int su[4] = {s4.x, s4.y, s4.z, s4.w};
        const int c = su[0] & 7;                         // source class, same for the 4 rows
        const double* ko = kb + (o * 64) * 2;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int sga = 2 * kk + (kq >> 1);
          const int aoff = 2 * (sga ^ c) + pk;
          double af[4], bf[2];
#pragma unroll
          for (int m = 0; m < 4; ++m) af[m] = q[su[m] * 16 + aoff];
#pragma unroll
          for (int jn = 0; jn < 2; ++jn) {
            const int tau = 4 * jn + (g8 >> 1);
            const double v = ko[(sga * 8 + (tau ^ ((sga & 1) << 1))) * 2 + comp];
            bf[jn] = __longlong_as_double(__double_as_longlong(v) ^ (long long)neg);
          }
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int jn = 0; jn < 2; ++jn) dmma_884(acc[m][jn], af[m], bf[jn]);
        }
      }
      C* pf = phat + (f0 + i) * ntc * 8 * nrhs + r;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        if (tgt[m] < 0) continue;
#pragma unroll
        for (int jn = 0; jn < 2; ++jn) {
          C* p = pf + ((cb + tgt[m]) * 8 + 4 * jn + kq) * nrhs;
          C v{acc[m][jn][0], acc[m][jn][1]};
          if (accumulate) {
            const C old = *p;
            v.x += old.x;
            v.y += old.y;
          }
          *p = v;
        }
      }
    }
    __syncthreads();
  }
}

template <typename T>
int hadamard_tiled(const T* khat, const T* qhat, const int64_t* tile_begin, const int64_t* src_off,
                   const int64_t* src, const int16_t* slots, const int16_t* tcol, int64_t n_tiles,
                   int64_t nf, int64_t nsc, int64_t ntc, int64_t nrhs, int accumulate, T* phat,
                   void* stream) {
  using C = typename cx<T>::v;
  if (n_tiles < 0 || nf < 0 || nsc < 0 || ntc < 0 || nrhs < 1 || nsc > INT32_MAX) return KIFMM_EARG;
  if (n_tiles == 0 || nf == 0) return 0;
  const size_t smem = (2 * 26 * 64 + 2 * QROWS * 8) * sizeof(C) + 26 * TT * sizeof(int16_t) +
                      UMAX * sizeof(int);
  dim3 grid((unsigned)n_tiles, ceil_div(nf, FCH), (unsigned)nrhs);
  if constexpr (sizeof(T) == 8) {
    {
      set_max_smem((const void*)hadamard_tiled_dmma_kernel, smem);
      hadamard_tiled_dmma_kernel<<<grid, 256, smem, (cudaStream_t)stream>>>(
          reinterpret_cast<const double2*>(khat), reinterpret_cast<const double2*>(qhat),
          tile_begin, src_off, src, slots, tcol, nf, nsc, ntc, nrhs, accumulate,
          reinterpret_cast<double2*>(phat));
      return launch_status();
    }
  }
  set_max_smem((const void*)hadamard_tiled_kernel<T>, smem);
  hadamard_tiled_kernel<T><<<grid, 256, smem, (cudaStream_t)stream>>>(
      reinterpret_cast<const C*>(khat), reinterpret_cast<const C*>(qhat), tile_begin, src_off, src,
      slots, tcol, nf, nsc, ntc, nrhs, accumulate, reinterpret_cast<C*>(phat));
  return launch_status();
}

}  // namespace

extern "C" {

int kifmm_hadamard_m2l_c64(const float* khat, const float* qhat, const int64_t* halo, float* phat,
                           int64_t nf, int64_t nsc, int64_t ntc, int64_t nrhs, void* s) {
  return hadamard<float>(khat, qhat, halo, phat, nf, nsc, ntc, nrhs, s);
}
int kifmm_hadamard_m2l_c128(const double* khat, const double* qhat, const int64_t* halo,
                            double* phat, int64_t nf, int64_t nsc, int64_t ntc, int64_t nrhs,
                            void* s) {
  return hadamard<double>(khat, qhat, halo, phat, nf, nsc, ntc, nrhs, s);
}

int kifmm_hadamard_tiled_c64(const float* khat, const float* qhat, const int64_t* tile_begin,
                             const int64_t* src_off, const int64_t* src, const int16_t* slots,
                             const int16_t* tcol, int64_t n_tiles, int64_t nf, int64_t nsc,
                             int64_t ntc, int64_t nrhs, int accumulate, float* phat, void* s) {
  return hadamard_tiled<float>(khat, qhat, tile_begin, src_off, src, slots, tcol, n_tiles, nf, nsc,
                               ntc, nrhs, accumulate, phat, s);
}
int kifmm_hadamard_tiled_c128(const double* khat, const double* qhat, const int64_t* tile_begin,
                              const int64_t* src_off, const int64_t* src, const int16_t* slots,
                              const int16_t* tcol, int64_t n_tiles, int64_t nf, int64_t nsc,
                              int64_t ntc, int64_t nrhs, int accumulate, double* phat, void* s) {
  return hadamard_tiled<double>(khat, qhat, tile_begin, src_off, src, slots, tcol, n_tiles, nf,
                                nsc, ntc, nrhs, accumulate, phat, s);
}

}  // extern "C"
