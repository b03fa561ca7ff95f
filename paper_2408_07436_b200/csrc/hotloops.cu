// Kernel-level plug-in boundary: device versions of the four loops of the
// reference's kifmm3d/_hot.pyx (bound through hotloops.py:54-77).
//
// Semantics kept from the reference:
//  * K(t, s) = (1/4pi)/|t - s|, zero when r2 == 0 (_hot.pyx:44-50);
//  * outputs accumulate (+=), laplace_matrix overwrites (_hot.pyx:68-88);
//  * per-target summation follows the source order (_hot.pyx:30-32);
//  * the fourth loop, hadamard_m2l (_hot.pyx:141-178), lives in hadamard.cu.
#include "common.cuh"

using namespace kifmm;

namespace {

constexpr int kTile = 256;

// One thread per target; sources staged through shared memory in tiles.
template <typename T>
__global__ void __launch_bounds__(kTile) potentials_kernel(
    const T* __restrict__ tx, const T* __restrict__ ty, const T* __restrict__ tz, int64_t nt,
    const T* __restrict__ sx, const T* __restrict__ sy, const T* __restrict__ sz, int64_t ns,
    const T* __restrict__ q, int64_t nrhs, T* __restrict__ out) {
  __shared__ T s_x[kTile], s_y[kTile], s_z[kTile];
  int64_t i = (int64_t)blockIdx.x * kTile + threadIdx.x;
  bool live = i < nt;
  T x = live ? tx[i] : T(0), y = live ? ty[i] : T(0), z = live ? tz[i] : T(0);
  for (int64_t r = 0; r < nrhs; ++r) {
    T acc = T(0);
    for (int64_t j0 = 0; j0 < ns; j0 += kTile) {
      int64_t j = j0 + threadIdx.x;
      __syncthreads();
      if (j < ns) { s_x[threadIdx.x] = sx[j]; s_y[threadIdx.x] = sy[j]; s_z[threadIdx.x] = sz[j]; }
      __syncthreads();
      int m = (int)min64(kTile, ns - j0);
      for (int jj = 0; jj < m; ++jj) {
        T w = inv_r<T>(x - s_x[jj], y - s_y[jj], z - s_z[jj]);
        acc += w * __ldg(&q[(j0 + jj) * nrhs + r]);
      }
    }
    if (live) out[i * nrhs + r] += acc * real_traits<T>::inv4pi();
  }
}

// Potential and gradient by direct summation (the gradient is an extension:
// the reference is potential-only; config 3 asks for both).  phi += sum q K,
// grad += sum q grad_t K = -sum q (t - s) / (4 pi r^3); r2 == 0 skipped.
template <typename T>
__global__ void __launch_bounds__(kTile) gradients_kernel(
    const T* __restrict__ tx, const T* __restrict__ ty, const T* __restrict__ tz, int64_t nt,
    const T* __restrict__ sx, const T* __restrict__ sy, const T* __restrict__ sz, int64_t ns,
    const T* __restrict__ q, int64_t nrhs, T* __restrict__ phi, T* __restrict__ grad) {
  __shared__ T s_x[kTile], s_y[kTile], s_z[kTile];
  int64_t i = (int64_t)blockIdx.x * kTile + threadIdx.x;
  bool live = i < nt;
  T x = live ? tx[i] : T(0), y = live ? ty[i] : T(0), z = live ? tz[i] : T(0);
  for (int64_t r = 0; r < nrhs; ++r) {
    T acc = T(0), gx = T(0), gy = T(0), gz = T(0);
    for (int64_t j0 = 0; j0 < ns; j0 += kTile) {
      int64_t j = j0 + threadIdx.x;
      __syncthreads();
      if (j < ns) { s_x[threadIdx.x] = sx[j]; s_y[threadIdx.x] = sy[j]; s_z[threadIdx.x] = sz[j]; }
      __syncthreads();
      int m = (int)min64(kTile, ns - j0);
      for (int jj = 0; jj < m; ++jj) {
        const T dx = x - s_x[jj], dy = y - s_y[jj], dz = z - s_z[jj];
        const T w = inv_r<T>(dx, dy, dz);
        const T qw = w * __ldg(&q[(j0 + jj) * nrhs + r]), qw3 = qw * w * w;
        acc += qw;
        gx -= dx * qw3; gy -= dy * qw3; gz -= dz * qw3;
      }
    }
    if (live) {
      const T c = real_traits<T>::inv4pi();
      phi[i * nrhs + r] += acc * c;
      T* g = grad + (i * nrhs + r) * 3;
      g[0] += gx * c; g[1] += gy * c; g[2] += gz * c;
    }
  }
}

// out[i, j] = fl(1/4pi) / sqrt(r2): IEEE division and square root, so the
// matrix is bit-identical to the reference's compiled loop.
template <typename T>
__global__ void matrix_kernel(const T* __restrict__ tx, const T* __restrict__ ty,
                              const T* __restrict__ tz, int64_t nt, const T* __restrict__ sx,
                              const T* __restrict__ sy, const T* __restrict__ sz, int64_t ns,
                              T* __restrict__ out) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nt * ns) return;
  int64_t i = idx / ns, j = idx - i * ns;
  T dx = tx[i] - sx[j], dy = ty[i] - sy[j], dz = tz[i] - sz[j];
  T r2 = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
  out[idx] = r2 > T(0) ? real_traits<T>::inv4pi() / sqrt(r2) : T(0);
}

template <>
__global__ void matrix_kernel<double>(const double* __restrict__ tx, const double* __restrict__ ty,
                                      const double* __restrict__ tz, int64_t nt,
                                      const double* __restrict__ sx, const double* __restrict__ sy,
                                      const double* __restrict__ sz, int64_t ns,
                                      double* __restrict__ out) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nt * ns) return;
  int64_t i = idx / ns, j = idx - i * ns;
  double dx = tx[i] - sx[j], dy = ty[i] - sy[j], dz = tz[i] - sz[j];
  double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  out[idx] = r2 > 0.0 ? KIFMM_INV_4PI_D / sqrt(r2) : 0.0;
}

// Reference CSR form: target i reads the gathered range of its leaf.
// Consecutive targets share a leaf, so source loads broadcast within a warp.
template <typename T>
__global__ void p2p_csr_kernel(const T* __restrict__ tx, const T* __restrict__ ty,
                               const T* __restrict__ tz, int64_t nt,
                               const int64_t* __restrict__ leaf_of_target,
                               const T* __restrict__ sx, const T* __restrict__ sy,
                               const T* __restrict__ sz, const T* __restrict__ q, int64_t nrhs,
                               const int64_t* __restrict__ off, T* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nt) return;
  int64_t b = leaf_of_target[i];
  int64_t j0 = off[b], j1 = off[b + 1];
  T x = tx[i], y = ty[i], z = tz[i];
  for (int64_t r = 0; r < nrhs; ++r) {
    T acc = T(0);
    for (int64_t j = j0; j < j1; ++j) {
      T w = inv_r<T>(x - __ldg(&sx[j]), y - __ldg(&sy[j]), z - __ldg(&sz[j]));
      acc += w * __ldg(&q[j * nrhs + r]);
    }
    out[i * nrhs + r] += acc * real_traits<T>::inv4pi();
  }
}

template <typename T>
int gradients(const T* tx, const T* ty, const T* tz, int64_t nt, const T* sx, const T* sy,
              const T* sz, int64_t ns, const T* q, int64_t nrhs, T* phi, T* grad, void* stream) {
  if (nt < 0 || ns < 0 || nrhs < 1) return KIFMM_EARG;
  if (nt == 0 || ns == 0) return 0;
  gradients_kernel<T><<<ceil_div(nt, kTile), kTile, 0, (cudaStream_t)stream>>>(
      tx, ty, tz, nt, sx, sy, sz, ns, q, nrhs, phi, grad);
  return launch_status();
}

template <typename T>
int potentials(const T* tx, const T* ty, const T* tz, int64_t nt, const T* sx, const T* sy,
               const T* sz, int64_t ns, const T* q, int64_t nrhs, T* out, void* stream) {
  if (nt < 0 || ns < 0 || nrhs < 1) return KIFMM_EARG;
  if (nt == 0 || ns == 0) return 0;
  potentials_kernel<T><<<ceil_div(nt, kTile), kTile, 0, (cudaStream_t)stream>>>(
      tx, ty, tz, nt, sx, sy, sz, ns, q, nrhs, out);
  return launch_status();
}

template <typename T>
int matrix(const T* tx, const T* ty, const T* tz, int64_t nt, const T* sx, const T* sy,
           const T* sz, int64_t ns, T* out, void* stream) {
  if (nt < 0 || ns < 0) return KIFMM_EARG;
  if (nt == 0 || ns == 0) return 0;
  matrix_kernel<T><<<ceil_div(nt * ns, 256), 256, 0, (cudaStream_t)stream>>>(tx, ty, tz, nt, sx,
                                                                             sy, sz, ns, out);
  return launch_status();
}

template <typename T>
int p2p(const T* tx, const T* ty, const T* tz, int64_t nt, const int64_t* lot, const T* sx,
        const T* sy, const T* sz, const T* q, int64_t nrhs, const int64_t* off, int64_t nl, T* out,
        void* stream) {
  if (nt < 0 || nl < 0 || nrhs < 1) return KIFMM_EARG;
  if (nt == 0) return 0;
  p2p_csr_kernel<T><<<ceil_div(nt, 128), 128, 0, (cudaStream_t)stream>>>(tx, ty, tz, nt, lot, sx,
                                                                         sy, sz, q, nrhs, off, out);
  return launch_status();
}

}  // namespace

extern "C" {

int kifmm_laplace_potentials_f32(const float* tx, const float* ty, const float* tz, int64_t nt,
                                 const float* sx, const float* sy, const float* sz, int64_t ns,
                                 const float* q, int64_t nrhs, float* out, void* s) {
  return potentials<float>(tx, ty, tz, nt, sx, sy, sz, ns, q, nrhs, out, s);
}
int kifmm_laplace_potentials_f64(const double* tx, const double* ty, const double* tz, int64_t nt,
                                 const double* sx, const double* sy, const double* sz, int64_t ns,
                                 const double* q, int64_t nrhs, double* out, void* s) {
  return potentials<double>(tx, ty, tz, nt, sx, sy, sz, ns, q, nrhs, out, s);
}
int kifmm_laplace_gradients_f32(const float* tx, const float* ty, const float* tz, int64_t nt,
                                const float* sx, const float* sy, const float* sz, int64_t ns,
                                const float* q, int64_t nrhs, float* phi, float* grad, void* s) {
  return gradients<float>(tx, ty, tz, nt, sx, sy, sz, ns, q, nrhs, phi, grad, s);
}
int kifmm_laplace_gradients_f64(const double* tx, const double* ty, const double* tz, int64_t nt,
                                const double* sx, const double* sy, const double* sz, int64_t ns,
                                const double* q, int64_t nrhs, double* phi, double* grad,
                                void* s) {
  return gradients<double>(tx, ty, tz, nt, sx, sy, sz, ns, q, nrhs, phi, grad, s);
}
int kifmm_laplace_matrix_f32(const float* tx, const float* ty, const float* tz, int64_t nt,
                             const float* sx, const float* sy, const float* sz, int64_t ns,
                             float* out, void* s) {
  return matrix<float>(tx, ty, tz, nt, sx, sy, sz, ns, out, s);
}
int kifmm_laplace_matrix_f64(const double* tx, const double* ty, const double* tz, int64_t nt,
                             const double* sx, const double* sy, const double* sz, int64_t ns,
                             double* out, void* s) {
  return matrix<double>(tx, ty, tz, nt, sx, sy, sz, ns, out, s);
}
int kifmm_p2p_blocked_f32(const float* tx, const float* ty, const float* tz, int64_t nt,
                          const int64_t* lot, const float* sx, const float* sy, const float* sz,
                          const float* q, int64_t nrhs, const int64_t* off, int64_t nl, float* out,
                          void* s) {
  return p2p<float>(tx, ty, tz, nt, lot, sx, sy, sz, q, nrhs, off, nl, out, s);
}
int kifmm_p2p_blocked_f64(const double* tx, const double* ty, const double* tz, int64_t nt,
                          const int64_t* lot, const double* sx, const double* sy, const double* sz,
                          const double* q, int64_t nrhs, const int64_t* off, int64_t nl,
                          double* out, void* s) {
  return p2p<double>(tx, ty, tz, nt, lot, sx, sy, sz, q, nrhs, off, nl, out, s);
}
int kifmm_sm_target(void) { return 100; }

}  // extern "C"
