/*
 * ORACLE - test infrastructure only (tests/, __graft_entry__.smoke(), the
 * cpu_baseline leg of bench.py).  Never linked into the product.
 *
 * C restatement of the four OpenMP loops of the reference's
 * pkg/src/kifmm3d/_hot.pyx, with the same arithmetic so that results are
 * bit-identical to the reference's compiled extension when built without
 * FMA contraction (gcc -O3 -fopenmp, default x86-64 target; see Makefile):
 *   laplace_potentials  _hot.pyx:24-65
 *   laplace_matrix      _hot.pyx:68-88
 *   p2p_blocked         _hot.pyx:91-138
 *   hadamard_m2l        _hot.pyx:141-178
 * The f32 kernel weight is (float)INV_4PI / sqrtf(r2) (_hot.pyx:46-49); the
 * f64 weight INV_4PI / sqrt(r2).  Coincident pairs contribute zero.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>

static const double INV_4PI = 0.079577471545947667884441881686257181;

#define DEF_POTENTIALS(T, SUF, WEIGHT)                                                          \
  void oracle_laplace_potentials_##SUF(const T* tx, const T* ty, const T* tz, int64_t nt,      \
                                       const T* sx, const T* sy, const T* sz, int64_t ns,      \
                                       const T* q, int64_t nrhs, T* out, int threads) {        \
    _Pragma("omp parallel for schedule(static) num_threads(threads)")                         \
    for (int64_t i = 0; i < nt; ++i) {                                                         \
      if (nrhs == 1) {                                                                         \
        T acc = 0;                                                                             \
        for (int64_t j = 0; j < ns; ++j) {                                                     \
          T dx = tx[i] - sx[j], dy = ty[i] - sy[j], dz = tz[i] - sz[j];                       \
          T r2 = dx * dx + dy * dy + dz * dz;                                                  \
          if (r2 > 0) acc = acc + (T)(WEIGHT) * q[j];                                          \
        }                                                                                      \
        out[i] += acc;                                                                         \
      } else {                                                                                 \
        for (int64_t j = 0; j < ns; ++j) {                                                     \
          T dx = tx[i] - sx[j], dy = ty[i] - sy[j], dz = tz[i] - sz[j];                       \
          T r2 = dx * dx + dy * dy + dz * dz;                                                  \
          if (r2 > 0) {                                                                        \
            T w = (T)(WEIGHT);                                                                 \
            for (int64_t r = 0; r < nrhs; ++r) out[i * nrhs + r] += w * q[j * nrhs + r];       \
          }                                                                                    \
        }                                                                                      \
      }                                                                                        \
    }                                                                                          \
  }

DEF_POTENTIALS(float, f32, (float)INV_4PI / sqrtf(r2))
DEF_POTENTIALS(double, f64, INV_4PI / sqrt(r2))

#define DEF_MATRIX(T, SUF, WEIGHT)                                                              \
  void oracle_laplace_matrix_##SUF(const T* tx, const T* ty, const T* tz, int64_t nt,          \
                                   const T* sx, const T* sy, const T* sz, int64_t ns, T* out,  \
                                   int threads) {                                              \
    _Pragma("omp parallel for schedule(static) num_threads(threads)")                         \
    for (int64_t i = 0; i < nt; ++i)                                                           \
      for (int64_t j = 0; j < ns; ++j) {                                                       \
        T dx = tx[i] - sx[j], dy = ty[i] - sy[j], dz = tz[i] - sz[j];                         \
        T r2 = dx * dx + dy * dy + dz * dz;                                                    \
        out[i * ns + j] = r2 > 0 ? (T)(WEIGHT) : (T)0;                                         \
      }                                                                                        \
  }

DEF_MATRIX(float, f32, (float)INV_4PI / sqrtf(r2))
DEF_MATRIX(double, f64, INV_4PI / sqrt(r2))

#define DEF_P2P(T, SUF, WEIGHT)                                                                 \
  void oracle_p2p_blocked_##SUF(const T* tx, const T* ty, const T* tz, int64_t nt,             \
                                const int64_t* leaf_of_target, const T* sx, const T* sy,       \
                                const T* sz, const T* q, int64_t nrhs, const int64_t* off,     \
                                T* out, int threads) {                                         \
    _Pragma("omp parallel for schedule(static) num_threads(threads)")                         \
    for (int64_t i = 0; i < nt; ++i) {                                                         \
      int64_t b = leaf_of_target[i];                                                           \
      int64_t j0 = off[b], j1 = off[b + 1];                                                    \
      if (nrhs == 1) {                                                                         \
        T acc = 0;                                                                             \
        for (int64_t j = j0; j < j1; ++j) {                                                    \
          T dx = tx[i] - sx[j], dy = ty[i] - sy[j], dz = tz[i] - sz[j];                       \
          T r2 = dx * dx + dy * dy + dz * dz;                                                  \
          if (r2 > 0) acc = acc + (T)(WEIGHT) * q[j];                                          \
        }                                                                                      \
        out[i] += acc;                                                                         \
      } else {                                                                                 \
        for (int64_t j = j0; j < j1; ++j) {                                                    \
          T dx = tx[i] - sx[j], dy = ty[i] - sy[j], dz = tz[i] - sz[j];                       \
          T r2 = dx * dx + dy * dy + dz * dz;                                                  \
          if (r2 > 0) {                                                                        \
            T w = (T)(WEIGHT);                                                                 \
            for (int64_t r = 0; r < nrhs; ++r) out[i * nrhs + r] += w * q[j * nrhs + r];       \
          }                                                                                    \
        }                                                                                      \
      }                                                                                        \
    }                                                                                          \
  }

DEF_P2P(float, f32, (float)INV_4PI / sqrtf(r2))
DEF_P2P(double, f64, INV_4PI / sqrt(r2))

/* khat (nf,26,8,8), qhat (nf,nsc,8,nrhs), halo (ntc,26), phat (nf,ntc,8,nrhs). */
#define DEF_HADAMARD(C, SUF)                                                                    \
  void oracle_hadamard_m2l_##SUF(const C* khat, const C* qhat, const int64_t* halo, C* phat,   \
                                 int64_t nf, int64_t nsc, int64_t ntc, int64_t nrhs,           \
                                 int threads) {                                                \
    _Pragma("omp parallel for schedule(static) num_threads(threads)")                         \
    for (int64_t f = 0; f < nf; ++f)                                                           \
      for (int64_t c = 0; c < ntc; ++c)                                                        \
        for (int o = 0; o < 26; ++o) {                                                         \
          int64_t s = halo[c * 26 + o];                                                        \
          if (s < 0) continue;                                                                 \
          for (int t = 0; t < 8; ++t)                                                          \
            for (int g = 0; g < 8; ++g) {                                                      \
              C k = khat[((f * 26 + o) * 8 + t) * 8 + g];                                      \
              for (int64_t r = 0; r < nrhs; ++r) {                                             \
                C* p = &phat[((f * ntc + c) * 8 + t) * nrhs + r];                              \
                *p = *p + k * qhat[((f * nsc + s) * 8 + g) * nrhs + r];                        \
              }                                                                                \
            }                                                                                  \
        }                                                                                      \
  }

DEF_HADAMARD(float complex, c64)
DEF_HADAMARD(double complex, c128)
