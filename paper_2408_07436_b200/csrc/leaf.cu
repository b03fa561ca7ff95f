// Leaf-level passes of evaluate (reference engine.py:298-319 and 377-404).
//
//  * p2m_check: check-surface potentials of every source leaf from its own
//    points (the P2M right-hand side, engine.py:305-318);
//  * leaf_pass: fused L2P (downward equivalent surface -> targets,
//    engine.py:377-389) + near-field P2P (_hot.pyx:91-138 via
//    engine.py:391-397) + the un-permute to caller order (engine.py:399-404).
//    The near field is walked as the reference orders it: the target's own
//    leaf first, then its neighbour leaves by Morton code; sources are read
//    in place from the tree-ordered arrays (no per-leaf duplication).
//    The gradient variant (config 3, "potential and gradient"; the reference
//    is potential-only) adds grad = sum q grad_t(1/(4 pi |t - s|)) over the
//    same L2P and P2P sources.
//
// Surface points are formed from a float64 leaf centre and float64 unit
// offsets with an exact add and one rounding, which reproduces the host's
// per-leaf surface arrays (engine.py:149-156) bit for bit.
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

using namespace kifmm;

namespace {

template <typename T> struct vec4;
template <> struct vec4<float> { using v = float4; };
template <> struct vec4<double> { using v = double4; };

// one warp (= one leaf) per CTA: a finished leaf frees its slot at once (config 3:
// gradient L2P 840 -> 707 us, P2M check 422 -> 385 us against 4-warp CTAs)
constexpr int kWarps = 1;

template <typename T>
__global__ void __launch_bounds__(32 * kWarps) p2m_check_kernel(
    const T* __restrict__ sx, const T* __restrict__ sy, const T* __restrict__ sz,
    const T* __restrict__ q, int64_t nrhs, const int32_t* __restrict__ leaf_start,
    const int32_t* __restrict__ leaf_count, int64_t n_leaves, const double* __restrict__ centers,
    const double* __restrict__ base, int64_t nc, T* __restrict__ phi) {
  using V = typename vec4<T>::v;
  __shared__ V buf[kWarps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t leaf = (int64_t)blockIdx.x * kWarps + w;
  if (leaf >= n_leaves) return;
  const int64_t s0 = leaf_start[leaf];
  const int cnt = leaf_count[leaf];
  const double cx = centers[leaf * 3], cy = centers[leaf * 3 + 1], cz = centers[leaf * 3 + 2];
  for (int64_t r = 0; r < nrhs; ++r) {
    for (int64_t c0 = 0; c0 < nc; c0 += 32) {
      const int64_t c = c0 + lane;
      T px = 0, py = 0, pz = 0;
      if (c < nc) {
        px = real_traits<T>::from_d(exact_add(cx, base[c * 3]));
        py = real_traits<T>::from_d(exact_add(cy, base[c * 3 + 1]));
        pz = real_traits<T>::from_d(exact_add(cz, base[c * 3 + 2]));
      }
      T acc = 0;
      for (int j0 = 0; j0 < cnt; j0 += 32) {
        __syncwarp();
        if (j0 + lane < cnt) {
          int64_t j = s0 + j0 + lane;
          buf[w][lane] = V{sx[j], sy[j], sz[j], q[j * nrhs + r]};
        }
        __syncwarp();
        const int m = min(32, cnt - j0);
        for (int k = 0; k < m; ++k) {
          V s = buf[w][k];
          acc += inv_r<T>(px - s.x, py - s.y, pz - s.z) * s.w;
        }
      }
      if (c < nc) phi[(leaf * nrhs + r) * nc + c] = acc * real_traits<T>::inv4pi();
    }
  }
}

// Near-field staging capacity per warp (sources), see leaf_pass_kernel.
template <typename T> struct cap_of { static constexpr int v = sizeof(T) == 4 ? 512 : 256; };

// Sum over staged sources [0, m): the first `guarded` entries may coincide
// with a target (they come from the target's own leaf), the rest cannot: two
// points in different leaves have distinct coordinates, and every leaf
// boundary lies >= 1 leaf side away from 0, so r2 cannot underflow either.
// GRAD also accumulates g -= (t - s) q / r^3 (the gradient of q / r at t).
template <typename T, bool TWO, bool GRAD>
__device__ __forceinline__ void near_sum(const typename vec4<T>::v* buf, int m, int guarded,
                                         T x0, T y0, T z0, T x1, T y1, T z1, T& a0, T& a1,
                                         T (&g0)[3], T (&g1)[3]) {
  using V = typename vec4<T>::v;
  int k = 0;
  for (; k < guarded; ++k) {
    V s = buf[k];
    if constexpr (GRAD) {
      const T dx = x0 - s.x, dy = y0 - s.y, dz = z0 - s.z;
      const T r2 = dx * dx + dy * dy + dz * dz;
      const T ri = r2 > T(0) ? real_traits<T>::rsq(r2) : T(0);
      const T w = ri * s.w, w3 = w * ri * ri;
      a0 += w;
      g0[0] -= dx * w3; g0[1] -= dy * w3; g0[2] -= dz * w3;
      if (TWO) {
        const T ex = x1 - s.x, ey = y1 - s.y, ez = z1 - s.z;
        const T q2 = ex * ex + ey * ey + ez * ez;
        const T qi = q2 > T(0) ? real_traits<T>::rsq(q2) : T(0);
        const T v = qi * s.w, v3 = v * qi * qi;
        a1 += v;
        g1[0] -= ex * v3; g1[1] -= ey * v3; g1[2] -= ez * v3;
      }
    } else {
      a0 += inv_r<T>(x0 - s.x, y0 - s.y, z0 - s.z) * s.w;
      if (TWO) a1 += inv_r<T>(x1 - s.x, y1 - s.y, z1 - s.z) * s.w;
    }
  }
  T b0 = 0, b1 = 0;
#pragma unroll 4
  for (; k < m; ++k) {
    V s = buf[k];
    T dx = x0 - s.x, dy = y0 - s.y, dz = z0 - s.z;
    const T ri = real_traits<T>::rsq(dx * dx + dy * dy + dz * dz);
    b0 += ri * s.w;
    if constexpr (GRAD) {
      const T w3 = ri * ri * ri * s.w;
      g0[0] -= dx * w3; g0[1] -= dy * w3; g0[2] -= dz * w3;
    }
    if (TWO) {
      T ex = x1 - s.x, ey = y1 - s.y, ez = z1 - s.z;
      const T qi = real_traits<T>::rsq(ex * ex + ey * ey + ez * ez);
      b1 += qi * s.w;
      if constexpr (GRAD) {
        const T v3 = qi * qi * qi * s.w;
        g1[0] -= ex * v3; g1[1] -= ey * v3; g1[2] -= ez * v3;
      }
    }
  }
  a0 += b0;
  a1 += b1;
}

// Copy one (x, y, z, q) source record global -> shared asynchronously.
template <typename T>
__device__ __forceinline__ void stage_src(typename vec4<T>::v* dst, const typename vec4<T>::v* src) {
  if constexpr (sizeof(T) == 4) {
    cp_async16(dst, src, true);
  } else {
    cp_async16(dst, src, true);
    cp_async16(reinterpret_cast<char*>(dst) + 16, reinterpret_cast<const char*>(src) + 16, true);
  }
}

// Leaf pass: one warp per target leaf, up to 64 targets per pass (lane and
// lane+32).  The near-field sources of the leaf - its own leaf first, then
// the neighbours by Morton code - are staged from the AoS source array into
// shared memory with cp.async, all segments in flight at once, then swept.
// GRAD: also the potential gradient, grad[(perm[i] * nrhs + r) * 3 + c]
// (L2P from the same downward equivalent densities + P2P gradient kernel).
template <typename T, bool GRAD>
__global__ void __launch_bounds__(32 * kWarps) leaf_pass_kernel(
    const T* __restrict__ tx, const T* __restrict__ ty, const T* __restrict__ tz,
    const int32_t* __restrict__ tstart, const int32_t* __restrict__ tcount, int64_t n_tleaves,
    const double* __restrict__ centers, const double* __restrict__ base, int64_t ne,
    const T* __restrict__ local, const typename vec4<T>::v* __restrict__ src4, int64_t ns,
    const int32_t* __restrict__ sstart, const int32_t* __restrict__ scount,
    const int32_t* __restrict__ near_off, const int32_t* __restrict__ near_leaf, int64_t nrhs,
    const int64_t* __restrict__ perm, int parts, T* __restrict__ out, T* __restrict__ grad) {
  using V = typename vec4<T>::v;
  constexpr int kCap = cap_of<T>::v;
  __shared__ __align__(16) V sbuf[kWarps][kCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  V* buf = sbuf[w];
  const int64_t b = (int64_t)blockIdx.x * kWarps + w;
  if (b >= n_tleaves) return;
  const int64_t t0 = tstart[b];
  const int tc = tcount[b];
  const double cx = centers[b * 3], cy = centers[b * 3 + 1], cz = centers[b * 3 + 2];
  const int n0 = near_off[b], n1 = near_off[b + 1];
  for (int tb = 0; tb < tc; tb += 64) {
    const bool two = tc - tb > 32;                 // warp-uniform
    const bool live0 = tb + lane < tc, live1 = tb + 32 + lane < tc;
    const int64_t i0 = t0 + tb + lane, i1 = i0 + 32;
    const T x0 = live0 ? tx[i0] : T(0), y0 = live0 ? ty[i0] : T(0), z0 = live0 ? tz[i0] : T(0);
    const T x1 = live1 ? tx[i1] : T(0), y1 = live1 ? ty[i1] : T(0), z1 = live1 ? tz[i1] : T(0);
    for (int64_t r = 0; r < nrhs; ++r) {
      T far0 = 0, far1 = 0, near0 = 0, near1 = 0;
      T gf0[3] = {0, 0, 0}, gf1[3] = {0, 0, 0}, gn0[3] = {0, 0, 0}, gn1[3] = {0, 0, 0};
      // L2P: downward equivalent densities of the leaf -> its targets.
      const T* loc = local + (b * nrhs + r) * ne;
      for (int64_t e0 = 0; (parts & 1) && e0 < ne; e0 += kCap) {
        const int m = (int)min64(kCap, ne - e0);
        __syncwarp();
        for (int k = lane; k < m; k += 32) {
          const int64_t e = e0 + k;
          buf[k] = V{real_traits<T>::from_d(exact_add(cx, base[e * 3])),
                     real_traits<T>::from_d(exact_add(cy, base[e * 3 + 1])),
                     real_traits<T>::from_d(exact_add(cz, base[e * 3 + 2])), loc[e]};
        }
        __syncwarp();
        if (two) near_sum<T, true, GRAD>(buf, m, m, x0, y0, z0, x1, y1, z1, far0, far1, gf0, gf1);
        else near_sum<T, false, GRAD>(buf, m, m, x0, y0, z0, x1, y1, z1, far0, far1, gf0, gf1);
      }
      // P2P: own leaf first, then neighbours in Morton order.
      if (parts & 2) {
        const V* srow = src4 + r * ns;
        int fill = 0;
        // bit 3 of parts: every record may coincide with a target (float32
        // rounding merged points of different leaves, checked at setup)
        int guarded = (parts & 8) ? INT_MAX : n1 > n0 ? scount[near_leaf[n0]] : 0;
        auto flush = [&]() {
          cp_async_commit();
          cp_async_wait<0>();
          __syncwarp();
          const int g = min(guarded, fill);
          if (two) near_sum<T, true, GRAD>(buf, fill, g, x0, y0, z0, x1, y1, z1, near0, near1, gn0, gn1);
          else near_sum<T, false, GRAD>(buf, fill, g, x0, y0, z0, x1, y1, z1, near0, near1, gn0, gn1);
          guarded -= g;
          fill = 0;
          __syncwarp();
        };
        __syncwarp();
        for (int n = n0; n < n1; ++n) {
          const int sl = near_leaf[n];
          const int64_t j0 = sstart[sl];
          const int jc = scount[sl];
          for (int jb = 0; jb < jc;) {
            if (fill == kCap) flush();
            const int m = min(jc - jb, kCap - fill);
            for (int k = lane; k < m; k += 32) stage_src<T>(buf + fill + k, srow + j0 + jb + k);
            fill += m;
            jb += m;
          }
        }
        if (fill) flush();
      }
      const T c = real_traits<T>::inv4pi();
      if (live0) {
        const int64_t row = (perm ? perm[i0] : i0) * nrhs + r;
        T* o = out + row;
        const T v = far0 * c + near0 * c;
        *o = (parts & 4) ? *o + v : v;
        if constexpr (GRAD) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            T* gp = grad + row * 3 + d;
            const T gv = gf0[d] * c + gn0[d] * c;
            *gp = (parts & 4) ? *gp + gv : gv;
          }
        }
      }
      if (two && live1) {
        const int64_t row = (perm ? perm[i1] : i1) * nrhs + r;
        T* o = out + row;
        const T v = far1 * c + near1 * c;
        *o = (parts & 4) ? *o + v : v;
        if constexpr (GRAD) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            T* gp = grad + row * 3 + d;
            const T gv = gf1[d] * c + gn1[d] * c;
            *gp = (parts & 4) ? *gp + gv : gv;
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// float32 leaf pass on packed FP32 (FFMA2/FADD2/FMUL2, sm_100's f32x2 ops).
// The scalar pass is issue-bound (~8 instructions per interaction); here two
// interactions share each vector instruction:
//  * leaves of <= 32 targets: a lane's target against a PAIR of sources,
//    staged as [xA xB yA yB zA zB qA qB] so two LDS.128 yield packed pairs;
//  * leaves of 33..64 targets: a PAIR of targets (lane, lane + 32) against
//    one source, its coordinates used as broadcast scalars (no moves).
// 9 vector/MUFU instructions per 2 interactions.  Same sources, order of
// traversal and guard semantics as leaf_pass_kernel (the sums are split
// into two interleaved partial sums, so rounding differs in the last bits).
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 up2(u64 v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// 1/sqrt of both halves; GUARD: 0 where r2 == 0 (coincident points).
template <bool GUARD>
__device__ __forceinline__ u64 rsq2(u64 r2) {
  const float2 v = up2(r2);
  float a = real_traits<float>::rsq(v.x), b = real_traits<float>::rsq(v.y);
  if (GUARD) {
    a = v.x > 0.f ? a : 0.f;
    b = v.y > 0.f ? b : 0.f;
  }
  return pk2(a, b);
}

#ifndef KIFMM_LEAF_MINB
#define KIFMM_LEAF_MINB 7      // leaf-pass CTAs per SM the register budget is sized for
#endif
#ifndef KIFMM_SRC_CAP
#define KIFMM_SRC_CAP 448
#endif
// Source records staged per warp (448 sources; a near field of ~810 sources
// takes two passes): 4 warps x 7 KB = 28 KB per CTA.
constexpr int kSrcCap = KIFMM_SRC_CAP;

__device__ __forceinline__ void fma2_acc(u64& acc, u64 a, u64 b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
// Sum over AoS source records s = start, start + stride, ... < ns of the
// lane's two targets (X, Y, Z packed pairs) against each source; records
// below `guard_n` may coincide with a target (r2 = 0 -> no contribution).
// One 16-byte shared load per source feeds two interactions; two
// accumulators alternate so consecutive sources do not serialise on one
// FFMA2 chain.
__device__ __forceinline__ void quad_sum(const float4* buf, int ns, int guard_n, int start,
                                         int stride, u64 X64, u64 Y64, u64 Z64, u64& acc64) {
  // float2 intrinsics (FADD2/FMUL2/FFMA2): the compiler keeps the packed
  // accumulators in place (no register moves per interaction)
  const float2 X = up2(X64), Y = up2(Y64), Z = up2(Z64);
  float2 acc = up2(acc64), acc2 = make_float2(0.f, 0.f);
  auto body = [&](int j, float2& a_, auto guard) {
    constexpr bool G = decltype(guard)::value;
    const float4 s = buf[j];                         // (x, y, z, q)
    const float2 dx = __fadd2_rn(X, make_float2(-s.x, -s.x));
    const float2 dy = __fadd2_rn(Y, make_float2(-s.y, -s.y));
    const float2 dz = __fadd2_rn(Z, make_float2(-s.z, -s.z));
    const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
    float w0 = real_traits<float>::rsq(r2.x), w1 = real_traits<float>::rsq(r2.y);
    if (G) {
      w0 = r2.x > 0.f ? w0 : 0.f;
      w1 = r2.y > 0.f ? w1 : 0.f;
    }
    a_ = __ffma2_rn(make_float2(w0, w1), make_float2(s.w, s.w), a_);
  };
  int j = start;
  for (; j < guard_n && j < ns; j += stride) body(j, acc, std::true_type{});
  for (; j + 3 * stride < ns; j += 4 * stride) {
    body(j, acc, std::false_type{});
    body(j + stride, acc2, std::false_type{});
    body(j + 2 * stride, acc, std::false_type{});
    body(j + 3 * stride, acc2, std::false_type{});
  }
  for (; j < ns; j += stride) body(j, acc, std::false_type{});
  acc64 = pk2(acc.x + acc2.x, acc.y + acc2.y);
}

__global__ void __launch_bounds__(32 * kWarps, KIFMM_LEAF_MINB) leaf_pass_x2_kernel(
    const float* __restrict__ tx, const float* __restrict__ ty, const float* __restrict__ tz,
    const int32_t* __restrict__ tstart, const int32_t* __restrict__ tcount, int64_t n_tleaves,
    const double* __restrict__ centers, const double* __restrict__ base, int64_t ne,
    const float* __restrict__ local, const float4* __restrict__ src4, int64_t ns,
    const int32_t* __restrict__ sstart, const int32_t* __restrict__ scount,
    const int32_t* __restrict__ near_off, const int32_t* __restrict__ near_leaf, int64_t nrhs,
    const int64_t* __restrict__ perm, int parts, float* __restrict__ out) {
  constexpr int kCap = kSrcCap;
  __shared__ __align__(16) float4 sbuf[kWarps][kCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4* buf = sbuf[w];
  const int64_t b = (int64_t)blockIdx.x * kWarps + w;
  if (b >= n_tleaves) return;
  const int64_t t0 = tstart[b];
  const int tc = tcount[b];
  const double cx = centers[b * 3], cy = centers[b * 3 + 1], cz = centers[b * 3 + 2];
  const int n0 = near_off[b], n1 = near_off[b + 1];
  // The near-field segments (<= 27 leaves) are looked up by all lanes at
  // once and broadcast with shuffles: no serial chain of dependent loads.
  int seg_start = 0, seg_cnt = 0;
  if (lane < n1 - n0) {
    const int sl = near_leaf[n0 + lane];
    seg_start = sstart[sl];
    seg_cnt = scount[sl];
  }
  // Passes of up to 32 targets, two per lane (the halves of the packed FP32
  // pairs).  A pass of n targets uses R = next power of two >= n/2 lanes per
  // source subset and f = 32 / R subsets: lane l serves targets l % R and
  // l % R + R over the sources j = l / R (mod f); the f partial sums are
  // combined with shuffles.  (A leaf of 30 targets: 16 lanes x 2 targets x
  // half the sources each; of 37: one such pass and a 5-target pass at an
  // 8-way source split.)
  for (int tb = 0; tb < tc; tb += 32) {
    const int n = min(32, tc - tb);
    const int h = (n + 1) >> 1;
    const int R = h <= 1 ? 1 : 1 << (32 - __clz(h - 1));
    const int f = 32 / R, sub = lane / R;
    const int ti = lane % R;
    const bool live0 = ti < n, live1 = ti + R < n;
    const int64_t ia = t0 + tb + (live0 ? ti : 0), ib = t0 + tb + (live1 ? ti + R : 0);
    const u64 X = pk2(tx[ia], tx[ib]), Y = pk2(ty[ia], ty[ib]), Z = pk2(tz[ia], tz[ib]);
    for (int64_t r = 0; r < nrhs; ++r) {
      u64 far = pk2(0.f, 0.f), near = pk2(0.f, 0.f);
      // L2P: downward equivalent densities of the leaf -> its targets.
      const float* loc = local + (b * nrhs + r) * ne;
      for (int64_t e0 = 0; (parts & 1) && e0 < ne; e0 += kCap) {
        const int m = (int)min64(kCap, ne - e0);
        __syncwarp();
        for (int k = lane; k < m; k += 32) {
          const int64_t e = e0 + k;
          buf[k] = make_float4(real_traits<float>::from_d(exact_add(cx, base[e * 3])),
                               real_traits<float>::from_d(exact_add(cy, base[e * 3 + 1])),
                               real_traits<float>::from_d(exact_add(cz, base[e * 3 + 2])), loc[e]);
        }
        __syncwarp();
        quad_sum(buf, m, 0, sub, f, X, Y, Z, far);
      }
      // P2P: own leaf first, then neighbours in Morton order.
      if (parts & 2) {
        const float4* srow = src4 + r * ns;
        int fill = 0;
        int guarded = (parts & 8) ? INT_MAX : __shfl_sync(0xffffffffu, seg_cnt, 0);
        auto flush = [&]() {
          cp_async_commit();
          cp_async_wait<0>();
          __syncwarp();
          const int g = min(guarded, fill);
          quad_sum(buf, fill, g, sub, f, X, Y, Z, near);
          guarded -= g;
          fill = 0;
          __syncwarp();
        };
        __syncwarp();
        for (int nn = 0; nn < n1 - n0; ++nn) {
          const int64_t j0 = __shfl_sync(0xffffffffu, seg_start, nn & 31);
          const int jc = __shfl_sync(0xffffffffu, seg_cnt, nn & 31);
          for (int jb = 0; jb < jc;) {
            if (fill == kCap) flush();
            const int m = min(jc - jb, kCap - fill);
            for (int k = lane; k < m; k += 32) cp_async16_ca(buf + fill + k, srow + j0 + jb + k, true);
            fill += m;
            jb += m;
          }
        }
        if (fill) flush();
      }
      const float c = real_traits<float>::inv4pi();
      const float2 fv = up2(far), nv = up2(near);
      float fa = fv.x, fb = fv.y, na = nv.x, nb = nv.y;
      // combine the f source subsets of each target
      for (int off = R; off < 32; off <<= 1) {
        fa += __shfl_xor_sync(0xffffffffu, fa, off);
        fb += __shfl_xor_sync(0xffffffffu, fb, off);
        na += __shfl_xor_sync(0xffffffffu, na, off);
        nb += __shfl_xor_sync(0xffffffffu, nb, off);
      }
      if (sub == 0) {
        if (live0) {
          const int64_t i = t0 + tb + ti;
          float* o = out + (perm ? perm[i] : i) * nrhs + r;
          const float v = fa * c + na * c;
          *o = (parts & 4) ? *o + v : v;
        }
        if (live1) {
          const int64_t i = t0 + tb + ti + R;
          float* o = out + (perm ? perm[i] : i) * nrhs + r;
          const float v = fb * c + nb * c;
          *o = (parts & 4) ? *o + v : v;
        }
      }
    }
  }
}

// L2P only (the final pass of the overlapped evaluate, after the P2P ran
// early): the same packed-FP32 target mapping as leaf_pass_x2_kernel without
// the near-field machinery, 8 warps per CTA and 0.9 KB of shared memory per
// warp, so many leaves are in flight at once (the pass is latency-bound:
// ~56 interactions per target).
// one warp (= one leaf) per CTA, 32 CTAs per SM: a warp that is done frees
// its slot at once (config 2: 43.5 us; 8-warp CTAs 53 us, 4-warp x 10: 47.6 us)
constexpr int kL2pWarps = 1;
__global__ void __launch_bounds__(32 * kL2pWarps, 32) l2p_x2_kernel(
    const float* __restrict__ tx, const float* __restrict__ ty, const float* __restrict__ tz,
    const int32_t* __restrict__ tstart, const int32_t* __restrict__ tcount, int64_t n_tleaves,
    const double* __restrict__ centers, const double* __restrict__ base, int ne,
    const float* __restrict__ local, int64_t nrhs, const int64_t* __restrict__ perm,
    int accumulate, const float* __restrict__ addend, float* __restrict__ out) {
  extern __shared__ __align__(16) float4 l2p_buf[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4* buf = l2p_buf + w * ne;
  const int64_t b = (int64_t)blockIdx.x * kL2pWarps + w;
  if (b >= n_tleaves) return;
  const int64_t t0 = tstart[b];
  const int tc = tcount[b];
  const double cx = centers[b * 3], cy = centers[b * 3 + 1], cz = centers[b * 3 + 2];
  for (int tb = 0; tb < tc; tb += 32) {
    const int n = min(32, tc - tb);
    const int h = (n + 1) >> 1;
    const int R = h <= 1 ? 1 : 1 << (32 - __clz(h - 1));
    const int f = 32 / R, sub = lane / R;
    const int ti = lane % R;
    const bool live0 = ti < n, live1 = ti + R < n;
    const int64_t ia = t0 + tb + (live0 ? ti : 0), ib = t0 + tb + (live1 ? ti + R : 0);
    const u64 X = pk2(tx[ia], tx[ib]), Y = pk2(ty[ia], ty[ib]), Z = pk2(tz[ia], tz[ib]);
    // output rows and, when accumulating, the values already there (the
    // near field): issued before the interaction loop so the un-permuting
    // scatter at the end carries no dependent global load
    const int64_t oa = perm ? perm[ia] : ia, ob = perm ? perm[ib] : ib;
    for (int64_t r = 0; r < nrhs; ++r) {
      const float* loc = local + (b * nrhs + r) * ne;
      // addend: the near-field totals in TREE order (coalesced, and no load
      // that depends on perm); else the values already in out (caller order)
      float pa = 0.f, pb = 0.f;
      if (sub == 0 && addend) {
        if (live0) pa = addend[ia * nrhs + r];
        if (live1) pb = addend[ib * nrhs + r];
      } else if (accumulate && sub == 0) {
        if (live0) pa = out[oa * nrhs + r];
        if (live1) pb = out[ob * nrhs + r];
      }
      __syncwarp();
      for (int k = lane; k < ne; k += 32)
        buf[k] = make_float4(real_traits<float>::from_d(exact_add(cx, base[k * 3])),
                             real_traits<float>::from_d(exact_add(cy, base[k * 3 + 1])),
                             real_traits<float>::from_d(exact_add(cz, base[k * 3 + 2])), loc[k]);
      __syncwarp();
      u64 acc = pk2(0.f, 0.f);
      quad_sum(buf, ne, 0, sub, f, X, Y, Z, acc);
      const float2 av = up2(acc);
      float fa = av.x, fb = av.y;
      for (int off = R; off < 32; off <<= 1) {
        fa += __shfl_xor_sync(0xffffffffu, fa, off);
        fb += __shfl_xor_sync(0xffffffffu, fb, off);
      }
      const float c = real_traits<float>::inv4pi();
      if (sub == 0) {
        if (live0) out[oa * nrhs + r] = (accumulate || addend) ? pa + fa * c : fa * c;
        if (live1) out[ob * nrhs + r] = (accumulate || addend) ? pb + fb * c : fb * c;
      }
    }
  }
}

// float32 P2M check potentials on packed FP32: every lane evaluates two
// check points (c, c + 32) of its leaf against the leaf's sources, staged
// once per warp (one 16-byte shared load feeds two interactions).
// (single-warp CTAs as for the L2P pass: 37 vs 40 us at config 2)
constexpr int kP2mWarps = 1;
__global__ void __launch_bounds__(32 * kP2mWarps, 32) p2m_check_x2_kernel(
    const float* __restrict__ sx, const float* __restrict__ sy, const float* __restrict__ sz,
    const float* __restrict__ q, int64_t nrhs, const int32_t* __restrict__ leaf_start,
    const int32_t* __restrict__ leaf_count, int64_t n_leaves, const double* __restrict__ centers,
    const double* __restrict__ base, int64_t nc, float* __restrict__ phi) {
  __shared__ __align__(16) float4 buf[kP2mWarps][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t leaf = (int64_t)blockIdx.x * kP2mWarps + w;
  if (leaf >= n_leaves) return;
  const int64_t s0 = leaf_start[leaf];
  const int cnt = leaf_count[leaf];
  const double cx = centers[leaf * 3], cy = centers[leaf * 3 + 1], cz = centers[leaf * 3 + 2];
  for (int64_t c0 = 0; c0 < nc; c0 += 64) {
    const int64_t ca = c0 + lane, cb = c0 + 32 + lane;
    auto pt = [&](int64_t c, double o, int d) {
      return c < nc ? real_traits<float>::from_d(exact_add(o, base[c * 3 + d])) : 0.f;
    };
    const float2 X = make_float2(pt(ca, cx, 0), pt(cb, cx, 0));
    const float2 Y = make_float2(pt(ca, cy, 1), pt(cb, cy, 1));
    const float2 Z = make_float2(pt(ca, cz, 2), pt(cb, cz, 2));
    for (int64_t r = 0; r < nrhs; ++r) {
      float2 acc = make_float2(0.f, 0.f), acc2 = make_float2(0.f, 0.f);
      for (int j0 = 0; j0 < cnt; j0 += 64) {
        const int m = min(64, cnt - j0);
        __syncwarp();
        for (int k = lane; k < m; k += 32) {
          const int64_t j = s0 + j0 + k;
          buf[w][k] = make_float4(sx[j], sy[j], sz[j], q[j * nrhs + r]);
        }
        __syncwarp();
        auto body = [&](int k, float2& a_) {
          const float4 v = buf[w][k];
          const float2 dx = __fadd2_rn(X, make_float2(-v.x, -v.x));
          const float2 dy = __fadd2_rn(Y, make_float2(-v.y, -v.y));
          const float2 dz = __fadd2_rn(Z, make_float2(-v.z, -v.z));
          const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
          float w0 = real_traits<float>::rsq(r2.x), w1 = real_traits<float>::rsq(r2.y);
          w0 = r2.x > 0.f ? w0 : 0.f;
          w1 = r2.y > 0.f ? w1 : 0.f;
          a_ = __ffma2_rn(make_float2(w0, w1), make_float2(v.w, v.w), a_);
        };
        int k = 0;
        for (; k + 1 < m; k += 2) {
          body(k, acc);
          body(k + 1, acc2);
        }
        if (k < m) body(k, acc);
      }
      const float c = real_traits<float>::inv4pi();
      if (ca < nc) phi[(leaf * nrhs + r) * nc + ca] = (acc.x + acc2.x) * c;
      if (cb < nc) phi[(leaf * nrhs + r) * nc + cb] = (acc.y + acc2.y) * c;
    }
  }
}

// AoS source records for the leaf pass: out[r*ns + j] = (x_j, y_j, z_j, q[j*nrhs + r]).
template <typename T>
__global__ void pack_sources_kernel(const T* __restrict__ sx, const T* __restrict__ sy,
                                    const T* __restrict__ sz, const T* __restrict__ q, int64_t ns,
                                    int64_t nrhs, typename vec4<T>::v* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ns * nrhs) return;
  const int64_t r = idx / ns, j = idx - r * ns;
  out[idx] = typename vec4<T>::v{sx[j], sy[j], sz[j], q[j * nrhs + r]};
}

template <typename T>
int p2m_check(const T* sx, const T* sy, const T* sz, const T* q, int64_t nrhs, const int32_t* ls,
              const int32_t* lc, int64_t nl, const double* centers, const double* base, int64_t nc,
              T* phi, void* stream) {
  if (nl < 0 || nc < 1 || nrhs < 1) return KIFMM_EARG;
  if (nl == 0) return 0;
  if constexpr (sizeof(T) == 4) {
    p2m_check_x2_kernel<<<ceil_div(nl, kP2mWarps), 32 * kP2mWarps, 0, (cudaStream_t)stream>>>(
        sx, sy, sz, q, nrhs, ls, lc, nl, centers, base, nc, phi);
    return launch_status();
  }
  p2m_check_kernel<T><<<ceil_div(nl, kWarps), 32 * kWarps, 0, (cudaStream_t)stream>>>(
      sx, sy, sz, q, nrhs, ls, lc, nl, centers, base, nc, phi);
  return launch_status();
}

template <typename T>
int leaf_pass(const T* tx, const T* ty, const T* tz, const int32_t* ts, const int32_t* tcnt,
              int64_t ntl, const double* centers, const double* base, int64_t ne, const T* local,
              const T* src4, int64_t ns, const int32_t* ss, const int32_t* sc, const int32_t* no,
              const int32_t* nlf, int64_t nrhs, const int64_t* perm, int parts, T* out,
              T* grad, void* stream) {
  if (ntl < 0 || ne < 1 || nrhs < 1 || parts < 1 || parts > 15 || ns < 0) return KIFMM_EARG;
  if (ntl == 0) return 0;
  const auto* s4 = reinterpret_cast<const typename vec4<T>::v*>(src4);
  if constexpr (sizeof(T) == 4) {
    if (!grad && !(parts & 2) && ne <= 256) {
      const size_t smem = (size_t)kL2pWarps * ne * sizeof(float4);
      l2p_x2_kernel<<<ceil_div(ntl, kL2pWarps), 32 * kL2pWarps, smem, (cudaStream_t)stream>>>(
          tx, ty, tz, ts, tcnt, ntl, centers, base, (int)ne, local, nrhs, perm, (parts & 4) != 0,
          nullptr, out);
      return launch_status();
    }
    if (!grad) {
      leaf_pass_x2_kernel<<<ceil_div(ntl, kWarps), 32 * kWarps, 0, (cudaStream_t)stream>>>(
          tx, ty, tz, ts, tcnt, ntl, centers, base, ne, local, s4, ns, ss, sc, no, nlf, nrhs,
          perm, parts, out);
      return launch_status();
    }
  }
  if (grad)
    leaf_pass_kernel<T, true><<<ceil_div(ntl, kWarps), 32 * kWarps, 0, (cudaStream_t)stream>>>(
        tx, ty, tz, ts, tcnt, ntl, centers, base, ne, local, s4, ns, ss, sc, no, nlf, nrhs, perm,
        parts, out, grad);
  else
    leaf_pass_kernel<T, false><<<ceil_div(ntl, kWarps), 32 * kWarps, 0, (cudaStream_t)stream>>>(
        tx, ty, tz, ts, tcnt, ntl, centers, base, ne, local, s4, ns, ss, sc, no, nlf, nrhs, perm,
        parts, out, nullptr);
  return launch_status();
}

template <typename T>
int pack_sources(const T* sx, const T* sy, const T* sz, const T* q, int64_t ns, int64_t nrhs,
                 T* out, void* stream) {
  if (ns < 0 || nrhs < 1) return KIFMM_EARG;
  if (ns == 0) return 0;
  pack_sources_kernel<T><<<ceil_div(ns * nrhs, 256), 256, 0, (cudaStream_t)stream>>>(
      sx, sy, sz, q, ns, nrhs, reinterpret_cast<typename vec4<T>::v*>(out));
  return launch_status();
}

}  // namespace

extern "C" {

int kifmm_p2m_check_f32(const float* sx, const float* sy, const float* sz, const float* q,
                        int64_t nrhs, const int32_t* ls, const int32_t* lc, int64_t nl,
                        const double* centers, const double* base, int64_t nc, float* phi,
                        void* s) {
  return p2m_check<float>(sx, sy, sz, q, nrhs, ls, lc, nl, centers, base, nc, phi, s);
}
int kifmm_p2m_check_f64(const double* sx, const double* sy, const double* sz, const double* q,
                        int64_t nrhs, const int32_t* ls, const int32_t* lc, int64_t nl,
                        const double* centers, const double* base, int64_t nc, double* phi,
                        void* s) {
  return p2m_check<double>(sx, sy, sz, q, nrhs, ls, lc, nl, centers, base, nc, phi, s);
}
int kifmm_leaf_pass_f32(const float* tx, const float* ty, const float* tz, const int32_t* ts,
                        const int32_t* tc, int64_t ntl, const double* centers, const double* base,
                        int64_t ne, const float* local, const float* src4, int64_t ns,
                        const int32_t* ss, const int32_t* sc, const int32_t* no,
                        const int32_t* nlf, int64_t nrhs, const int64_t* perm, int parts,
                        float* out, void* s) {
  return leaf_pass<float>(tx, ty, tz, ts, tc, ntl, centers, base, ne, local, src4, ns, ss, sc, no,
                          nlf, nrhs, perm, parts, out, nullptr, s);
}
// L2P + addend: out[perm[i]] = addend[i] + L2P(i), addend in tree order (the
// near-field totals of kifmm_p2p_mutual_reduce_f32 with perm = NULL).
int kifmm_l2p_add_f32(const float* tx, const float* ty, const float* tz, const int32_t* ts,
                      const int32_t* tc, int64_t ntl, const double* centers, const double* base,
                      int64_t ne, const float* local, int64_t nrhs, const int64_t* perm,
                      const float* addend, float* out, void* s) {
  if (ntl < 0 || ne < 1 || ne > 256 || nrhs < 1 || !addend) return KIFMM_EARG;
  if (ntl == 0) return 0;
  const size_t smem = (size_t)kL2pWarps * ne * sizeof(float4);
  l2p_x2_kernel<<<ceil_div(ntl, kL2pWarps), 32 * kL2pWarps, smem, (cudaStream_t)s>>>(
      tx, ty, tz, ts, tc, ntl, centers, base, (int)ne, local, nrhs, perm, 0, addend, out);
  return launch_status();
}
int kifmm_leaf_pass_f64(const double* tx, const double* ty, const double* tz, const int32_t* ts,
                        const int32_t* tc, int64_t ntl, const double* centers, const double* base,
                        int64_t ne, const double* local, const double* src4, int64_t ns,
                        const int32_t* ss, const int32_t* sc, const int32_t* no,
                        const int32_t* nlf, int64_t nrhs, const int64_t* perm, int parts,
                        double* out, void* s) {
  return leaf_pass<double>(tx, ty, tz, ts, tc, ntl, centers, base, ne, local, src4, ns, ss, sc,
                           no, nlf, nrhs, perm, parts, out, nullptr, s);
}
int kifmm_leaf_pass_grad_f32(const float* tx, const float* ty, const float* tz, const int32_t* ts,
                             const int32_t* tc, int64_t ntl, const double* centers,
                             const double* base, int64_t ne, const float* local, const float* src4,
                             int64_t ns, const int32_t* ss, const int32_t* sc, const int32_t* no,
                             const int32_t* nlf, int64_t nrhs, const int64_t* perm, int parts,
                             float* out, float* grad, void* s) {
  if (!grad) return KIFMM_EARG;
  return leaf_pass<float>(tx, ty, tz, ts, tc, ntl, centers, base, ne, local, src4, ns, ss, sc, no,
                          nlf, nrhs, perm, parts, out, grad, s);
}
int kifmm_leaf_pass_grad_f64(const double* tx, const double* ty, const double* tz,
                             const int32_t* ts, const int32_t* tc, int64_t ntl,
                             const double* centers, const double* base, int64_t ne,
                             const double* local, const double* src4, int64_t ns,
                             const int32_t* ss, const int32_t* sc, const int32_t* no,
                             const int32_t* nlf, int64_t nrhs, const int64_t* perm, int parts,
                             double* out, double* grad, void* s) {
  if (!grad) return KIFMM_EARG;
  return leaf_pass<double>(tx, ty, tz, ts, tc, ntl, centers, base, ne, local, src4, ns, ss, sc,
                           no, nlf, nrhs, perm, parts, out, grad, s);
}
int kifmm_pack_sources_f32(const float* sx, const float* sy, const float* sz, const float* q,
                           int64_t ns, int64_t nrhs, float* out, void* s) {
  return pack_sources<float>(sx, sy, sz, q, ns, nrhs, out, s);
}
int kifmm_pack_sources_f64(const double* sx, const double* sy, const double* sz, const double* q,
                           int64_t ns, int64_t nrhs, double* out, void* s) {
  return pack_sources<double>(sx, sy, sz, q, ns, nrhs, out, s);
}
}  // extern "C"
