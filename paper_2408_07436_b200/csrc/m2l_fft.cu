// FFT-M2L transforms (replace the scipy.fft/numpy staging of reference
// m2l_fft.m2l_fft_level, m2l_fft.py:236-261).
//
// The multipole of a box occupies only the surface of the p^3 corner
// sub-cube [p, 2p)^3 of the n = 2p grid, and only the surface of [0, p)^3
// is read back after the inverse.  Both transforms are therefore done as
// three pruned 1-D DFT passes (one per axis) in shared memory:
//   forward: z (real->half complex, p inputs), y (p inputs), x (p inputs)
//   inverse: x (n inputs -> p outputs), y (n -> p), z (half complex -> p reals)
// One CTA handles one sibling cluster (8 boxes) so the frequency-major
// spectrum rows (f, cluster, child) are written/read 8 children at a time.
#include <cstdlib>

#include "common.cuh"

using namespace kifmm;

namespace {

template <typename T> struct cx;
template <> struct cx<float> { using v = float2; };
template <> struct cx<double> { using v = double2; };

template <typename C>
__device__ __forceinline__ C cmul(C a, C b) {
  return C{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename C>
__device__ __forceinline__ void cfma(C& acc, C a, C b) {
  acc.x += a.x * b.x - a.y * b.y;
  acc.y += a.x * b.y + a.y * b.x;
}

// Threads per CTA: the y pass has bpc * P * (P + 1) work items (576 at p = 8
// with 8 boxes per CTA) and the x pass twice that, so the block is sized to
// that count rounded up to a warp (one round of the y pass, two of the x
// pass), within [128, kMaxThreads].  (config 3 level 5 with 512 threads:
// forward 670 us; 256: 1000 us; 1024 spills: 700 / 1160 us; 4 or 2 boxes
// per CTA for more CTAs per SM: slower)
constexpr int kMaxThreads = 640;
constexpr size_t kSmemLimit = 227 * 1024;
// Boxes per CTA: the largest of 8/4/2/1 whose scratch fits (0: none).
constexpr int boxes_per_cta(size_t head, size_t box) {
  for (int bpc = 8; bpc >= 1; bpc /= 2)
    if (head + bpc * box <= kSmemLimit) return bpc;
  return 0;
}
constexpr int fft_threads(int bpc, int p) {
  const int t = (bpc * p * (p + 1) + 31) / 32 * 32;
  return t < 128 ? 128 : (t > kMaxThreads ? kMaxThreads : t);
}
constexpr int kMaxP = 12;

// Surface lattice of the p^3 cube in lexicographic order -> flat index
// (i*p + j)*p + k, built by one warp with ballots (reference
// expansion.py:34-42 ordering).
__device__ void build_lattice(int p, int* lat) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  int base = 0;
  const int p3 = p * p * p;
  for (int i0 = 0; i0 < p3; i0 += 32) {
    const int idx = i0 + lane;
    bool on = false;
    if (idx < p3) {
      int a = idx / (p * p), b = (idx / p) % p, c = idx % p;
      on = a == 0 || a == p - 1 || b == 0 || b == p - 1 || c == 0 || c == p - 1;
    }
    unsigned m = __ballot_sync(0xffffffffu, on);
    if (on) lat[base + __popc(m & ((1u << lane) - 1u))] = idx;
    base += __popc(m);
  }
}

// Twiddle table TW[k][m] = e^{-2 pi i (k m mod n) / n}, k, m < n: with the
// order a template constant every DFT loop below is unrolled and a twiddle
// read is (row base + immediate).
template <typename T>
__device__ void build_twiddles(int n, typename cx<T>::v* tw) {
  // the n roots once (row k = 1 of the table), then the table by index: one
  // sincospi per root instead of one per entry
  for (int m = threadIdx.x; m < n; m += blockDim.x) {
    double s, c;
    sincospi(2.0 * m / n, &s, &c);
    tw[n + m] = typename cx<T>::v{(T)c, (T)(-s)};
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int k = e / n, m = e % n;
    if (k != 1) tw[e] = tw[n + (k * m) % n];
  }
}

// Per-box scratch strides are padded to (multiple of 128 B) + sizeof(C) so
// the 8 boxes a warp's lanes touch at the same offset sit in 8 different
// bank groups.
template <typename C>
constexpr size_t pad_box(size_t bytes) {
  return ((bytes + 127) / 128) * 128 + sizeof(C);
}

template <typename T, int P>
struct FftShape {
  using C = typename cx<T>::v;
  static constexpr int N = 2 * P, NH = P + 1, NE = 6 * (P - 1) * (P - 1) + 2, P3 = P * P * P;
  static constexpr size_t head = ((N * N * sizeof(C) + NE * sizeof(int) + 127) / 128) * 128;
  // forward: X1 [P][P][NH] complex, then CUBE [P^3] real / X2 [P][N][NH] complex
  static constexpr size_t fx1 = (size_t)P * P * NH * sizeof(C);
  static constexpr size_t fu = (size_t)P * N * NH * sizeof(C) > (size_t)P3 * sizeof(T)
                                   ? (size_t)P * N * NH * sizeof(C) : (size_t)P3 * sizeof(T);
  static constexpr size_t fbox = pad_box<C>(fx1 + fu);
  // inverse: Y1 [P][N][NH], Y2 [P][P][NH]
  static constexpr size_t iy1 = (size_t)P * N * NH * sizeof(C);
  static constexpr size_t ibox = pad_box<C>(iy1 + (size_t)P * P * NH * sizeof(C));
  static constexpr int fbpc = boxes_per_cta(head, fbox), ibpc = boxes_per_cta(head, ibox);
  static constexpr int fthreads = fft_threads(fbpc ? fbpc : 1, P);
  static constexpr int ithreads = fft_threads(ibpc ? ibpc : 1, P);
};

template <typename T, int P>
__global__ void __launch_bounds__(FftShape<T, P>::fthreads) fft_forward_kernel(const T* __restrict__ mult,
                                                               int64_t nrhs, int bpc,
                                                               const int32_t* __restrict__ slot_box,
                                                               int64_t nsc,
                                                               const int32_t* __restrict__ cluster_list,
                                                               typename cx<T>::v* __restrict__ qhat) {
  using S = FftShape<T, P>;
  using C = typename cx<T>::v;
  constexpr int N = S::N, NH = S::NH, NE = S::NE, P3 = S::P3;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* tw = reinterpret_cast<C*>(smem_raw);
  int* lat = reinterpret_cast<int*>(smem_raw + N * N * sizeof(C));
  unsigned char* boxes = smem_raw + S::head;
  auto X1 = [&](int b) { return reinterpret_cast<C*>(boxes + b * S::fbox); };
  auto CUBE = [&](int b) { return reinterpret_cast<T*>(boxes + b * S::fbox + S::fx1); };
  auto X2 = [&](int b) { return reinterpret_cast<C*>(boxes + b * S::fbox + S::fx1); };

  const int groups = 8 / bpc;
  const int64_t cluster = cluster_list ? (int64_t)cluster_list[blockIdx.x / groups]
                                       : (int64_t)(blockIdx.x / groups);
  const int child0 = (blockIdx.x % groups) * bpc;
  const int64_t r = blockIdx.y;
  build_twiddles<T>(N, tw);
  build_lattice(P, lat);
  for (int e = threadIdx.x; e < bpc * P3; e += (int)blockDim.x) CUBE(e % bpc)[e / bpc] = T(0);
  __syncthreads();
  for (int e = threadIdx.x; e < bpc * NE; e += (int)blockDim.x) {
    const int b = e / NE, s = e - b * NE;
    const int32_t box = slot_box[cluster * 8 + child0 + b];
    if (box >= 0) CUBE(b)[lat[s]] = mult[((int64_t)box * nrhs + r) * NE + s];
  }
  __syncthreads();
  // z: X1[i0][i1][k2] = sum_{i2} cube[i0][i1][i2] w^{k2 (i2 + P)}; thread per line.
  for (int e = threadIdx.x; e < bpc * P * P; e += (int)blockDim.x) {
    const int b = e % bpc, i01 = e / bpc;
    T line[P];
#pragma unroll
    for (int i2 = 0; i2 < P; ++i2) line[i2] = CUBE(b)[i01 * P + i2];
    C* out = X1(b) + i01 * NH;
#pragma unroll 2
    for (int k2 = 0; k2 < NH; ++k2) {
      const C* w = tw + k2 * N + P;
      C acc{0, 0};
#pragma unroll
      for (int i2 = 0; i2 < P; ++i2) {
        acc.x = fma(line[i2], w[i2].x, acc.x);
        acc.y = fma(line[i2], w[i2].y, acc.y);
      }
      out[k2] = acc;
    }
  }
  __syncthreads();
  // y: X2[i0][k1][k2] = sum_{i1} X1[i0][i1][k2] w^{k1 (i1 + P)} (overwrites the cube).
  for (int e = threadIdx.x; e < bpc * P * NH; e += (int)blockDim.x) {
    const int b = e % bpc, rem = e / bpc;
    const int k2 = rem % NH, i0 = rem / NH;
    C in[P];
#pragma unroll
    for (int i1 = 0; i1 < P; ++i1) in[i1] = X1(b)[(i0 * P + i1) * NH + k2];
#pragma unroll 2
    for (int k1 = 0; k1 < N; ++k1) {
      const C* w = tw + k1 * N + P;
      C acc{0, 0};
#pragma unroll
      for (int i1 = 0; i1 < P; ++i1) cfma(acc, in[i1], w[i1]);
      X2(b)[(i0 * N + k1) * NH + k2] = acc;
    }
  }
  __syncthreads();
  // x: spectrum[k0][k1][k2] = sum_{i0} X2[i0][k1][k2] w^{k0 (i0 + P)}, child fastest.
  for (int e = threadIdx.x; e < N * NH * bpc; e += (int)blockDim.x) {
    const int b = e % bpc, k12 = e / bpc;
    C in[P];
#pragma unroll
    for (int i0 = 0; i0 < P; ++i0) in[i0] = X2(b)[i0 * N * NH + k12];
    C* dst = qhat + (((int64_t)k12 * nsc + cluster) * 8 + child0 + b) * nrhs + r;
    const int64_t fstride = (int64_t)N * NH * nsc * 8 * nrhs;
#pragma unroll 2
    for (int k0 = 0; k0 < N; ++k0) {
      const C* w = tw + k0 * N + P;
      C acc{0, 0};
#pragma unroll
      for (int i0 = 0; i0 < P; ++i0) cfma(acc, in[i0], w[i0]);
      dst[k0 * fstride] = acc;
    }
  }
}

template <typename T, int P>
__global__ void __launch_bounds__(FftShape<T, P>::ithreads) fft_inverse_kernel(const typename cx<T>::v* __restrict__ phat,
                                                               int64_t nrhs, int bpc,
                                                               const int32_t* __restrict__ slot_box,
                                                               int64_t ntc, T scale,
                                                               T* __restrict__ check) {
  using S = FftShape<T, P>;
  using C = typename cx<T>::v;
  constexpr int N = S::N, NH = S::NH, NE = S::NE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* tw = reinterpret_cast<C*>(smem_raw);
  int* lat = reinterpret_cast<int*>(smem_raw + N * N * sizeof(C));
  unsigned char* boxes = smem_raw + S::head;
  auto Y1 = [&](int b) { return reinterpret_cast<C*>(boxes + b * S::ibox); };
  auto Y2 = [&](int b) { return reinterpret_cast<C*>(boxes + b * S::ibox + S::iy1); };

  const int groups = 8 / bpc;
  const int64_t cluster = blockIdx.x / groups;
  const int child0 = (blockIdx.x % groups) * bpc;
  const int64_t r = blockIdx.y;
  build_twiddles<T>(N, tw);
  build_lattice(P, lat);
  __syncthreads();
  // x: Y1[i0][k1][k2] = sum_{k0} X[k0][k1][k2] w^{-k0 i0}, i0 < P; child fastest.
  for (int e = threadIdx.x; e < N * NH * bpc; e += (int)blockDim.x) {
    const int b = e % bpc, k12 = e / bpc;
    const C* src = phat + (((int64_t)k12 * ntc + cluster) * 8 + child0 + b) * nrhs + r;
    const int64_t fstride = (int64_t)N * NH * ntc * 8 * nrhs;
    C in[N];
#pragma unroll
    for (int k0 = 0; k0 < N; ++k0) in[k0] = src[k0 * fstride];
#pragma unroll 2
    for (int i0 = 0; i0 < P; ++i0) {
      C acc{0, 0};
#pragma unroll
      for (int k0 = 0; k0 < N; ++k0) {
        const C w = tw[i0 * N + k0];           // conj(w) applied below
        acc.x = fma(in[k0].x, w.x, fma(in[k0].y, w.y, acc.x));
        acc.y = fma(in[k0].y, w.x, fma(-in[k0].x, w.y, acc.y));
      }
      Y1(b)[i0 * N * NH + k12] = acc;
    }
  }
  __syncthreads();
  // y: Y2[i0][i1][k2] = sum_{k1} Y1[i0][k1][k2] w^{-k1 i1}, i1 < P.
  for (int e = threadIdx.x; e < P * NH * bpc; e += (int)blockDim.x) {
    const int b = e % bpc, rem = e / bpc;
    const int k2 = rem % NH, i0 = rem / NH;
    C in[N];
#pragma unroll
    for (int k1 = 0; k1 < N; ++k1) in[k1] = Y1(b)[(i0 * N + k1) * NH + k2];
#pragma unroll 2
    for (int i1 = 0; i1 < P; ++i1) {
      C acc{0, 0};
#pragma unroll
      for (int k1 = 0; k1 < N; ++k1) {
        const C w = tw[i1 * N + k1];
        acc.x = fma(in[k1].x, w.x, fma(in[k1].y, w.y, acc.x));
        acc.y = fma(in[k1].y, w.x, fma(-in[k1].x, w.y, acc.y));
      }
      Y2(b)[(i0 * P + i1) * NH + k2] = acc;
    }
  }
  __syncthreads();
  // z (complex -> real, Hermitian half spectrum; the imaginary parts of the
  // k2 = 0 and Nyquist bins are ignored as in pocketfft's c2r), read the
  // lattice, normalise by n^3 and apply the level scale.
  const T norm = T(1) / (T)(N * N * N);
  for (int e = threadIdx.x; e < NE * bpc; e += (int)blockDim.x) {
    const int b = e % bpc, s = e / bpc;
    const int32_t box = slot_box[cluster * 8 + child0 + b];
    if (box < 0) continue;
    const int li = lat[s];
    const int i01 = li / P, i2 = li - i01 * P;
    const C* y = Y2(b) + i01 * NH;
    const C* w = tw + i2 * N;                  // Re(y e^{+i theta}) = y.x cos + y.y (-sin)
    T acc = y[0].x + ((i2 & 1) ? -y[P].x : y[P].x);
    T mid = 0;
#pragma unroll
    for (int k2 = 1; k2 < P; ++k2) mid = fma(y[k2].x, w[k2].x, fma(y[k2].y, w[k2].y, mid));
    acc += T(2) * mid;
    check[((int64_t)box * nrhs + r) * NE + s] = (acc * norm) * scale;
  }
}

template <typename T, int P>
size_t forward_smem(int bpc) { return FftShape<T, P>::head + bpc * FftShape<T, P>::fbox; }
template <typename T, int P>
size_t inverse_smem(int bpc) { return FftShape<T, P>::head + bpc * FftShape<T, P>::ibox; }

template <typename T, int P>
int forward_p(const T* mult, int64_t nrhs, const int32_t* slot_box, int64_t nsc,
              const int32_t* cluster_list, int64_t nclusters, T* qhat, cudaStream_t stream) {
  using C = typename cx<T>::v;
  constexpr int bpc = FftShape<T, P>::fbpc;
  if (!bpc) return KIFMM_EARG;
  const size_t smem = forward_smem<T, P>(bpc);
  set_max_smem((const void*)fft_forward_kernel<T, P>, smem);
  dim3 grid((unsigned)(nclusters * (8 / bpc)), (unsigned)nrhs);
  fft_forward_kernel<T, P><<<grid, FftShape<T, P>::fthreads, smem, stream>>>(
      mult, nrhs, bpc, slot_box, nsc, cluster_list, reinterpret_cast<C*>(qhat));
  return launch_status();
}

template <typename T, int P>
int inverse_p(const T* phat, int64_t nrhs, const int32_t* slot_box, int64_t ntc, double scale,
              T* check, cudaStream_t stream) {
  using C = typename cx<T>::v;
  constexpr int bpc = FftShape<T, P>::ibpc;
  if (!bpc) return KIFMM_EARG;
  const size_t smem = inverse_smem<T, P>(bpc);
  set_max_smem((const void*)fft_inverse_kernel<T, P>, smem);
  dim3 grid((unsigned)(ntc * (8 / bpc)), (unsigned)nrhs);
  fft_inverse_kernel<T, P><<<grid, FftShape<T, P>::ithreads, smem, stream>>>(
      reinterpret_cast<const C*>(phat), nrhs, bpc, slot_box, ntc, (T)scale, check);
  return launch_status();
}

#define KIFMM_ORDERS(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12)

template <typename T>
int forward(const T* mult, int64_t nrhs, int64_t order, const int32_t* slot_box, int64_t nsc,
            const int32_t* cluster_list, int64_t n_list, T* qhat, void* stream) {
  if (order < 2 || order > kMaxP || nrhs < 1 || nsc < 0) return KIFMM_EARG;
  if (nsc == 0) return 0;
  const int64_t nclusters = cluster_list ? n_list : nsc;
  if (nclusters <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  switch (order) {
#define X(P_) case P_: return forward_p<T, P_>(mult, nrhs, slot_box, nsc, cluster_list, nclusters, qhat, s);
    KIFMM_ORDERS(X)
#undef X
  }
  return KIFMM_EARG;
}

template <typename T>
int inverse(const T* phat, int64_t nrhs, int64_t order, const int32_t* slot_box, int64_t ntc,
            double level_scale, T* check, void* stream) {
  if (order < 2 || order > kMaxP || nrhs < 1 || ntc < 0) return KIFMM_EARG;
  if (ntc == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  switch (order) {
#define X(P_) case P_: return inverse_p<T, P_>(phat, nrhs, slot_box, ntc, level_scale, check, s);
    KIFMM_ORDERS(X)
#undef X
  }
  return KIFMM_EARG;
}

}  // namespace

extern "C" {

int kifmm_fft_forward_f32(const float* mult, int64_t nrhs, int64_t order, const int32_t* slot_box,
                          int64_t nsc, const int32_t* cluster_list, int64_t n_list, float* qhat,
                          void* s) {
  return forward<float>(mult, nrhs, order, slot_box, nsc, cluster_list, n_list, qhat, s);
}
int kifmm_fft_forward_f64(const double* mult, int64_t nrhs, int64_t order,
                          const int32_t* slot_box, int64_t nsc, const int32_t* cluster_list,
                          int64_t n_list, double* qhat, void* s) {
  return forward<double>(mult, nrhs, order, slot_box, nsc, cluster_list, n_list, qhat, s);
}
int kifmm_fft_inverse_f32(const float* phat, int64_t nrhs, int64_t order, const int32_t* slot_box,
                          int64_t ntc, double level_scale, float* check, void* s) {
  return inverse<float>(phat, nrhs, order, slot_box, ntc, level_scale, check, s);
}
int kifmm_fft_inverse_f64(const double* phat, int64_t nrhs, int64_t order,
                          const int32_t* slot_box, int64_t ntc, double level_scale, double* check,
                          void* s) {
  return inverse<double>(phat, nrhs, order, slot_box, ntc, level_scale, check, s);
}

}  // extern "C"
