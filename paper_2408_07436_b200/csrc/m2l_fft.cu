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

constexpr int kThreads = 256;
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

template <typename T>
__device__ void build_twiddles(int n, typename cx<T>::v* tw) {
  for (int m = threadIdx.x; m < n; m += blockDim.x) {
    double s, c;
    sincospi(2.0 * m / n, &s, &c);
    tw[m] = typename cx<T>::v{(T)c, (T)(-s)};   // e^{-2 pi i m / n}
  }
}

template <typename T>
size_t forward_smem(int p, int bpc) {
  using C = typename cx<T>::v;
  int n = 2 * p, nh = p + 1, ne = 6 * (p - 1) * (p - 1) + 2;
  size_t per_box_x1 = (size_t)p * p * nh * sizeof(C);
  size_t cube = (size_t)p * p * p * sizeof(T);
  size_t x2 = (size_t)p * n * nh * sizeof(C);
  size_t per_box = per_box_x1 + (cube > x2 ? cube : x2);
  return n * sizeof(C) + ((ne * sizeof(int) + 15) / 16) * 16 + bpc * per_box;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) fft_forward_kernel(const T* __restrict__ mult,
                                                               int64_t nrhs, int p, int bpc,
                                                               const int32_t* __restrict__ slot_box,
                                                               int64_t nsc,
                                                               const int32_t* __restrict__ cluster_list,
                                                               typename cx<T>::v* __restrict__ qhat) {
  using C = typename cx<T>::v;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = 2 * p, nh = p + 1, ne = 6 * (p - 1) * (p - 1) + 2, p3 = p * p * p;
  C* tw = reinterpret_cast<C*>(smem_raw);
  int* lat = reinterpret_cast<int*>(smem_raw + n * sizeof(C));
  unsigned char* boxes = smem_raw + n * sizeof(C) + ((ne * sizeof(int) + 15) / 16) * 16;
  const size_t x1_elems = (size_t)p * p * nh;
  const size_t u_bytes = max((size_t)p3 * sizeof(T), (size_t)p * n * nh * sizeof(C));
  const size_t box_bytes = x1_elems * sizeof(C) + u_bytes;
  auto X1 = [&](int b) { return reinterpret_cast<C*>(boxes + b * box_bytes); };
  auto CUBE = [&](int b) { return reinterpret_cast<T*>(boxes + b * box_bytes + x1_elems * sizeof(C)); };
  auto X2 = [&](int b) { return reinterpret_cast<C*>(boxes + b * box_bytes + x1_elems * sizeof(C)); };

  const int groups = 8 / bpc;
  const int64_t cluster = cluster_list ? (int64_t)cluster_list[blockIdx.x / groups]
                                       : (int64_t)(blockIdx.x / groups);
  const int child0 = (blockIdx.x % groups) * bpc;
  const int64_t r = blockIdx.y;
  build_twiddles<T>(n, tw);
  build_lattice(p, lat);
  for (int e = threadIdx.x; e < bpc * p3; e += kThreads) CUBE(e / p3)[e % p3] = T(0);
  __syncthreads();
  for (int e = threadIdx.x; e < bpc * ne; e += kThreads) {
    const int b = e / ne, s = e - b * ne;
    const int32_t box = slot_box[cluster * 8 + child0 + b];
    if (box >= 0) CUBE(b)[lat[s]] = mult[((int64_t)box * nrhs + r) * ne + s];
  }
  __syncthreads();
  // z: X1[i0][i1][k2] = sum_{i2} cube[i0][i1][i2] w^{k2 (i2 + p)}
  for (int e = threadIdx.x; e < bpc * p * p * nh; e += kThreads) {
    const int b = e / (p * p * nh);
    int rem = e - b * p * p * nh;
    const int k2 = rem % nh, i01 = rem / nh;
    const T* line = CUBE(b) + i01 * p;
    C acc{0, 0};
    for (int i2 = 0; i2 < p; ++i2) {
      C w = tw[(k2 * (i2 + p)) % n];
      acc.x += line[i2] * w.x;
      acc.y += line[i2] * w.y;
    }
    X1(b)[i01 * nh + k2] = acc;
  }
  __syncthreads();
  // y: X2[i0][k1][k2] = sum_{i1} X1[i0][i1][k2] w^{k1 (i1 + p)}   (overwrites the cube)
  for (int e = threadIdx.x; e < bpc * p * n * nh; e += kThreads) {
    const int b = e / (p * n * nh);
    int rem = e - b * p * n * nh;
    const int k2 = rem % nh, k1 = (rem / nh) % n, i0 = rem / (nh * n);
    C acc{0, 0};
    for (int i1 = 0; i1 < p; ++i1) cfma(acc, X1(b)[(i0 * p + i1) * nh + k2], tw[(k1 * (i1 + p)) % n]);
    X2(b)[(i0 * n + k1) * nh + k2] = acc;
  }
  __syncthreads();
  // x: spectrum[k0][k1][k2] = sum_{i0} X2[i0][k1][k2] w^{k0 (i0 + p)}, child fastest
  const int nf = n * n * nh;
  for (int e = threadIdx.x; e < nf * bpc; e += kThreads) {
    const int b = e % bpc, f = e / bpc;
    const int k0 = f / (n * nh), k12 = f % (n * nh);
    C acc{0, 0};
    for (int i0 = 0; i0 < p; ++i0) cfma(acc, X2(b)[i0 * n * nh + k12], tw[(k0 * (i0 + p)) % n]);
    qhat[(((int64_t)f * nsc + cluster) * 8 + child0 + b) * nrhs + r] = acc;
  }
}

template <typename T>
size_t inverse_smem(int p, int bpc) {
  using C = typename cx<T>::v;
  int n = 2 * p, nh = p + 1, ne = 6 * (p - 1) * (p - 1) + 2;
  size_t y1 = (size_t)p * n * nh * sizeof(C), y2 = (size_t)p * p * nh * sizeof(C);
  return n * sizeof(C) + ((ne * sizeof(int) + 15) / 16) * 16 + bpc * (y1 + y2);
}

template <typename T>
__global__ void __launch_bounds__(kThreads) fft_inverse_kernel(const typename cx<T>::v* __restrict__ phat,
                                                               int64_t nrhs, int p, int bpc,
                                                               const int32_t* __restrict__ slot_box,
                                                               int64_t ntc, T scale,
                                                               T* __restrict__ check) {
  using C = typename cx<T>::v;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = 2 * p, nh = p + 1, ne = 6 * (p - 1) * (p - 1) + 2;
  C* tw = reinterpret_cast<C*>(smem_raw);
  int* lat = reinterpret_cast<int*>(smem_raw + n * sizeof(C));
  unsigned char* boxes = smem_raw + n * sizeof(C) + ((ne * sizeof(int) + 15) / 16) * 16;
  const size_t y1e = (size_t)p * n * nh, y2e = (size_t)p * p * nh;
  auto Y1 = [&](int b) { return reinterpret_cast<C*>(boxes) + b * (y1e + y2e); };
  auto Y2 = [&](int b) { return reinterpret_cast<C*>(boxes) + b * (y1e + y2e) + y1e; };

  const int groups = 8 / bpc;
  const int64_t cluster = blockIdx.x / groups;
  const int child0 = (blockIdx.x % groups) * bpc;
  const int64_t r = blockIdx.y;
  build_twiddles<T>(n, tw);
  build_lattice(p, lat);
  __syncthreads();
  // x: Y1[i0][k1][k2] = sum_{k0} X[k0][k1][k2] w^{-k0 i0}, i0 < p; child fastest.
  for (int e = threadIdx.x; e < n * nh * bpc; e += kThreads) {
    const int b = e % bpc, k12 = e / bpc;
    C acc[kMaxP];
#pragma unroll
    for (int i = 0; i < kMaxP; ++i) acc[i] = C{0, 0};
    for (int k0 = 0; k0 < n; ++k0) {
      const int64_t f = (int64_t)k0 * n * nh + k12;
      const C v = phat[((f * ntc + cluster) * 8 + child0 + b) * nrhs + r];
#pragma unroll
      for (int i0 = 0; i0 < kMaxP; ++i0) {
        if (i0 < p) {
          C w = tw[(k0 * i0) % n];
          w.y = -w.y;
          cfma(acc[i0], v, w);
        }
      }
    }
#pragma unroll
    for (int i0 = 0; i0 < kMaxP; ++i0)
      if (i0 < p) Y1(b)[i0 * n * nh + k12] = acc[i0];
  }
  __syncthreads();
  // y: Y2[i0][i1][k2] = sum_{k1} Y1[i0][k1][k2] w^{-k1 i1}, i1 < p.
  for (int e = threadIdx.x; e < p * nh * bpc; e += kThreads) {
    const int b = e % bpc, rem = e / bpc;
    const int k2 = rem % nh, i0 = rem / nh;
    C acc[kMaxP];
#pragma unroll
    for (int i = 0; i < kMaxP; ++i) acc[i] = C{0, 0};
    for (int k1 = 0; k1 < n; ++k1) {
      const C v = Y1(b)[(i0 * n + k1) * nh + k2];
#pragma unroll
      for (int i1 = 0; i1 < kMaxP; ++i1) {
        if (i1 < p) {
          C w = tw[(k1 * i1) % n];
          w.y = -w.y;
          cfma(acc[i1], v, w);
        }
      }
    }
#pragma unroll
    for (int i1 = 0; i1 < kMaxP; ++i1)
      if (i1 < p) Y2(b)[(i0 * p + i1) * nh + k2] = acc[i1];
  }
  __syncthreads();
  // z (complex -> real, Hermitian half spectrum; the imaginary parts of the
  // k2 = 0 and Nyquist bins are ignored as in pocketfft's c2r), read the
  // lattice, normalise by n^3 and apply the level scale.
  const T norm = T(1) / (T)(n * n * n);
  for (int e = threadIdx.x; e < ne * bpc; e += kThreads) {
    const int b = e % bpc, s = e / bpc;
    const int32_t box = slot_box[cluster * 8 + child0 + b];
    if (box < 0) continue;
    const int li = lat[s];
    const int i0 = li / (p * p), i1 = (li / p) % p, i2 = li % p;
    const C* y = Y2(b) + (i0 * p + i1) * nh;
    T acc = y[0].x + ((i2 & 1) ? -y[p].x : y[p].x);
    T mid = 0;
    for (int k2 = 1; k2 < p; ++k2) {
      C w = tw[(k2 * i2) % n];   // e^{-i theta}; Re(y e^{+i theta}) = y.x cos + y.y (-sin)
      mid += y[k2].x * w.x + y[k2].y * w.y;
    }
    acc += T(2) * mid;
    check[((int64_t)box * nrhs + r) * ne + s] = (acc * norm) * scale;
  }
}

int pick_bpc(size_t (*smem)(int, int), int p, size_t limit) {
  for (int bpc = 8; bpc >= 1; bpc /= 2)
    if (smem(p, bpc) <= limit) return bpc;
  return 0;
}

template <typename T>
int forward(const T* mult, int64_t nrhs, int64_t order, const int32_t* slot_box, int64_t nsc,
            const int32_t* cluster_list, int64_t n_list, T* qhat, void* stream) {
  using C = typename cx<T>::v;
  if (order < 2 || order > kMaxP || nrhs < 1 || nsc < 0) return KIFMM_EARG;
  if (nsc == 0) return 0;
  const int p = (int)order;
  const int bpc = pick_bpc(forward_smem<T>, p, 227 * 1024);
  if (!bpc) return KIFMM_EARG;
  size_t smem = forward_smem<T>(p, bpc);
  auto kern = fft_forward_kernel<T>;
  set_max_smem((const void*)kern, smem);
  const int64_t nclusters = cluster_list ? n_list : nsc;
  if (nclusters <= 0) return 0;
  dim3 grid((unsigned)(nclusters * (8 / bpc)), (unsigned)nrhs);
  kern<<<grid, kThreads, smem, (cudaStream_t)stream>>>(mult, nrhs, p, bpc, slot_box, nsc,
                                                       cluster_list, reinterpret_cast<C*>(qhat));
  return launch_status();
}

template <typename T>
int inverse(const T* phat, int64_t nrhs, int64_t order, const int32_t* slot_box, int64_t ntc,
            double level_scale, T* check, void* stream) {
  using C = typename cx<T>::v;
  if (order < 2 || order > kMaxP || nrhs < 1 || ntc < 0) return KIFMM_EARG;
  if (ntc == 0) return 0;
  const int p = (int)order;
  const int bpc = pick_bpc(inverse_smem<T>, p, 227 * 1024);
  if (!bpc) return KIFMM_EARG;
  size_t smem = inverse_smem<T>(p, bpc);
  auto kern = fft_inverse_kernel<T>;
  set_max_smem((const void*)kern, smem);
  dim3 grid((unsigned)(ntc * (8 / bpc)), (unsigned)nrhs);
  kern<<<grid, kThreads, smem, (cudaStream_t)stream>>>(reinterpret_cast<const C*>(phat), nrhs, p,
                                                       bpc, slot_box, ntc, (T)level_scale, check);
  return launch_status();
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
