// Mutual (symmetric) near field for sources == targets, potential (float32 on
// packed FP32 pairs, float64 on the FP64 pipe: the same kernel, templated).
//
// The reference's P2P (_hot.pyx:91-138 over the gather plan of
// engine.py:224-256) evaluates, for every target leaf A, K(t_i, s_j) for all
// points j of A and of its adjacent leaves.  When the source and target
// clouds are the same point set, each pair of adjacent leaves (A, B) is met
// twice - once from A's side, once from B's - with the same 1/r.  Here every
// unordered pair of distinct adjacent leaves is evaluated ONCE, by the lower
// leaf A (leaf rows are in Morton order): one rsqrt feeds both directions,
//   phi_i += q_j / r_ij   (row sums, A's targets, in registers)
//   psi_j += q_i / r_ij   (column sums, B's targets),
// halving the MUFU work (the P2P bound).  The leaf's own block (A, A) keeps
// the direct form, with the r2 = 0 guard (coincident points contribute 0,
// _hot.pyx:44-50).
//
// Determinism without atomics: every partial sum has ONE writer and a fixed
// place.  The partial buffer P holds, per target leaf B (n_B points,
// nlow_B adjacent leaves below B in Morton order),
//   slot 0            B's own row sums (self block + all upper pairs)
//   slot s = 1..nlow  the column sums contributed by the s-th lower
//                     neighbour (B's near list is [B, neighbours ascending],
//                     so the lower neighbours are entries 1..nlow)
// at P[base_B + s n_B + t]; mutual_reduce_kernel adds the slots of each
// target in slot order into the caller-ordered output (un-permuted,
// engine.py:399-404) and the L2P pass accumulates the far field onto it.
//
// Column sums inside a warp: a pass holds up to 32 targets of A, two per
// lane (packed FP32 pairs, as leaf_pass_x2_kernel), in f = 32 / R groups of
// R lanes; the upper neighbours' points are concatenated into columns and
// each group takes chunks of R columns.  Lane t of a group meets column
// (t + s) mod R at step s; its column accumulator psi moves one lane down
// after every step (one shuffle per half), so after R steps lane t holds the
// complete column sum of column t.  Each chunk is staged twice in a row in
// shared memory, so the wrap needs no index arithmetic (a load at an
// immediate offset per step).  Per step: 1 LDS.128, 3 FADD2, FMUL2, 2 FFMA2
// (r2), 2 MUFU.RSQ, 2 FFMA2 (row, column), 2 SHFL - for 4 interactions.
//
// Precondition of the unguarded upper blocks: no two points of DIFFERENT
// leaves coincide after rounding to float32 (checked at setup; the guarded
// variant is launched otherwise).
#include <cstdlib>

#include "common.cuh"

using namespace kifmm;

namespace {

#ifndef KIFMM_MUT_WARPS
#define KIFMM_MUT_WARPS 2
#endif
// warps per CTA (one target leaf per warp): single-warp CTAs release their
// resources as soon as their leaf is done (the work per leaf varies with its
// count of upper neighbours, 0..26)
constexpr int kMW = KIFMM_MUT_WARPS;
#ifndef KIFMM_MUT_MINB
#define KIFMM_MUT_MINB (20 / KIFMM_MUT_WARPS)   // CTAs per SM the register budget is sized for
#endif
constexpr unsigned kFull = 0xffffffffu;

// Pairs of targets: float -> packed FP32 (FADD2 / FMUL2 / FFMA2), double ->
// two scalars.
template <typename T> struct pr;
template <> struct pr<float> {
  using P2 = float2;
  using Rec = float4;
  static __device__ __forceinline__ P2 mk(float a, float b) { return make_float2(a, b); }
  static __device__ __forceinline__ P2 add(P2 a, P2 b) { return __fadd2_rn(a, b); }
  static __device__ __forceinline__ P2 mul(P2 a, P2 b) { return __fmul2_rn(a, b); }
  static __device__ __forceinline__ P2 fma(P2 a, P2 b, P2 c) { return __ffma2_rn(a, b, c); }
  // pad coordinate: finite (inf - x = inf would put 0 * inf = NaN into the
  // gradient sums); r2 = 3e36, w ~ 6e-19 times the pad's zero charge = 0, w^3
  // underflows to 0, and the pad's own column sums are never stored
  static __device__ __forceinline__ float inf() { return 1e18f; }
  static constexpr int kFC = 128;                 // columns per fill
};
template <> struct pr<double> {
  using P2 = double2;
  using Rec = double4;
  static __device__ __forceinline__ P2 mk(double a, double b) { return make_double2(a, b); }
  static __device__ __forceinline__ P2 add(P2 a, P2 b) { return make_double2(a.x + b.x, a.y + b.y); }
  static __device__ __forceinline__ P2 mul(P2 a, P2 b) { return make_double2(a.x * b.x, a.y * b.y); }
  static __device__ __forceinline__ P2 fma(P2 a, P2 b, P2 c) {
    return make_double2(::fma(a.x, b.x, c.x), ::fma(a.y, b.y, c.y));
  }
  // (finite as well - the Newton steps of the float64 rsqrt turn inf * 0 into
  // NaN: r2 = 3e300, w ~ 6e-151, w^3 underflows to 0)
  static __device__ __forceinline__ double inf() { return 1e150; }
  static constexpr int kFC = 64;                  // 32-byte records: the same bytes per fill
};

template <typename T>
__device__ __forceinline__ typename pr<T>::Rec pad_col() {
  // far-away, chargeless: no contribution either way
  typename pr<T>::Rec c;
  c.x = c.y = c.z = pr<T>::inf();
  c.w = T(0);
  return c;
}
template <typename T>
__device__ __forceinline__ void cp_async_rec(typename pr<T>::Rec* dst, const typename pr<T>::Rec* src) {
  cp_async16(dst, src, true);
  if (sizeof(T) == 8)
    cp_async16(reinterpret_cast<char*>(dst) + 16, reinterpret_cast<const char*>(src) + 16, true);
}

// Row-only sum over staged records [0, m) for the lane's four targets (two
// pairs: X0 = targets (0, 1), X1 = (2, 3)), sources j = start,
// start + stride, ...; every record may coincide with a target (the leaf's
// own block): r2 = 0 contributes 0.
template <typename T>
struct Quad {
  typename pr<T>::P2 X0, Y0, Z0, X1, Y1, Z1;
};
// Differences and squared distance of a pair of targets to one record.
template <typename T>
struct Diff {
  typename pr<T>::P2 dx, dy, dz, r2;
};
template <typename T>
__device__ __forceinline__ Diff<T> diff2(typename pr<T>::P2 X, typename pr<T>::P2 Y,
                                         typename pr<T>::P2 Z, const typename pr<T>::Rec& s) {
  using O = pr<T>;
  Diff<T> d;
  d.dx = O::add(X, O::mk(-s.x, -s.x));
  d.dy = O::add(Y, O::mk(-s.y, -s.y));
  d.dz = O::add(Z, O::mk(-s.z, -s.z));
  d.r2 = O::fma(d.dz, d.dz, O::fma(d.dy, d.dy, O::mul(d.dx, d.dx)));
  return d;
}
template <typename T, bool GUARD>
__device__ __forceinline__ typename pr<T>::P2 rsq2f(typename pr<T>::P2 r2) {
  T w0 = real_traits<T>::rsq(r2.x), w1 = real_traits<T>::rsq(r2.y);
  if (GUARD) {
    w0 = r2.x > T(0) ? w0 : T(0);
    w1 = r2.y > T(0) ? w1 : T(0);
  }
  return pr<T>::mk(w0, w1);
}

// Row sums of the lane's four targets: the potential and, with GRAD, G =
// sum_j q_j (t - s_j) / r^3 per component (the gradient of the potential is
// -G; the sign is applied when the sums are written).
template <typename T>
struct Rows {
  typename pr<T>::P2 phi0, phi1, g0x, g0y, g0z, g1x, g1y, g1z;
};
// Column sums of one column: psi = sum_i q_i / r and, with GRAD, H = sum_i q_i
// (t_i - s) / r^3 (the gradient of the potential at the column point is +H).
template <typename T>
struct Cols {
  typename pr<T>::P2 psi, hx, hy, hz;
};

template <typename T, bool GUARD, bool GRAD, bool COLS>
__device__ __forceinline__ void pair_step(const Quad<T>& t, const typename pr<T>::Rec& c,
                                          typename pr<T>::P2 QA0, typename pr<T>::P2 QA1,
                                          Rows<T>& a, Cols<T>& h) {
  using O = pr<T>;
  const Diff<T> d0 = diff2<T>(t.X0, t.Y0, t.Z0, c), d1 = diff2<T>(t.X1, t.Y1, t.Z1, c);
  const auto w0 = rsq2f<T, GUARD>(d0.r2), w1 = rsq2f<T, GUARD>(d1.r2);
  const auto q = O::mk(c.w, c.w);
  a.phi0 = O::fma(w0, q, a.phi0);
  a.phi1 = O::fma(w1, q, a.phi1);
  if (COLS) h.psi = O::fma(w1, QA1, O::fma(w0, QA0, h.psi));
  if (GRAD) {
    const auto c0 = O::mul(O::mul(w0, w0), w0), c1 = O::mul(O::mul(w1, w1), w1);   // 1 / r^3
    const auto r0 = O::mul(q, c0), r1 = O::mul(q, c1);
    a.g0x = O::fma(r0, d0.dx, a.g0x);
    a.g0y = O::fma(r0, d0.dy, a.g0y);
    a.g0z = O::fma(r0, d0.dz, a.g0z);
    a.g1x = O::fma(r1, d1.dx, a.g1x);
    a.g1y = O::fma(r1, d1.dy, a.g1y);
    a.g1z = O::fma(r1, d1.dz, a.g1z);
    if (COLS) {
      const auto k0 = O::mul(QA0, c0), k1 = O::mul(QA1, c1);
      h.hx = O::fma(k1, d1.dx, O::fma(k0, d0.dx, h.hx));
      h.hy = O::fma(k1, d1.dy, O::fma(k0, d0.dy, h.hy));
      h.hz = O::fma(k1, d1.dz, O::fma(k0, d0.dz, h.hz));
    }
  }
}

// Row-only sum over staged records [0, m) for the lane's four targets (two
// pairs: X0 = targets (0, 1), X1 = (2, 3)), sources j = start,
// start + stride, ...; every record may coincide with a target (the leaf's
// own block): r2 = 0 contributes 0.
template <typename T, bool GRAD>
__device__ __forceinline__ void self_sum(const typename pr<T>::Rec* buf, int m, int start,
                                         int stride, const Quad<T>& t, Rows<T>& a) {
  Cols<T> none;
  const auto z = pr<T>::mk(T(0), T(0));
  for (int j = start; j < m; j += stride)
    pair_step<T, true, GRAD, false>(t, buf[j], z, z, a, none);
}

// Rounds of 32 staged columns (f chunks of R); group grp takes chunk
// round * f + grp.  Chunk k occupies buf[2Rk, 2Rk + 2R) (the chunk twice).
// Per step a lane meets one column with its four targets: one record load
// and two shuffles (eight with GRAD) feed four interactions.  Pr: the
// right-hand side's first component plane; cstride: elements between the
// component planes (potential, then the three gradient components).
template <typename T, int R, bool GUARD, bool GRAD>
__device__ __forceinline__ void mutual_rounds(const typename pr<T>::Rec* buf, const int32_t* dst,
                                              int m, int grp, int ti, const Quad<T>& t,
                                              typename pr<T>::P2 QA0, typename pr<T>::P2 QA1,
                                              Rows<T>& a, T* __restrict__ Pr, int64_t cstride,
                                              bool rmw) {
  using O = pr<T>;
  constexpr int NC = GRAD ? 4 : 1;
  for (int c0 = 0; c0 < m; c0 += 32) {
    const int k = c0 / R + grp;                    // R is a compile-time power of two
    const typename O::Rec* p = buf + 2 * R * k + ti;
    const int col = k * R + ti;
    // a later target pass of the same leaf adds to the column sums of the
    // earlier ones: fetch them before the chain of steps
    T* o = Pr + (col < m ? dst[col] : 0);
    T old[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) old[c] = (rmw && col < m) ? __ldcg(o + c * cstride) : T(0);
    Cols<T> h;
    h.psi = h.hx = h.hy = h.hz = O::mk(T(0), T(0));
#pragma unroll
    for (int s = 0; s < R; ++s) {
      pair_step<T, GUARD, GRAD, true>(t, p[s], QA0, QA1, a, h);
      if (R > 1) {
        h.psi.x = __shfl_sync(kFull, h.psi.x, ti + 1, R);
        h.psi.y = __shfl_sync(kFull, h.psi.y, ti + 1, R);
        if (GRAD) {
          h.hx.x = __shfl_sync(kFull, h.hx.x, ti + 1, R);
          h.hx.y = __shfl_sync(kFull, h.hx.y, ti + 1, R);
          h.hy.x = __shfl_sync(kFull, h.hy.x, ti + 1, R);
          h.hy.y = __shfl_sync(kFull, h.hy.y, ti + 1, R);
          h.hz.x = __shfl_sync(kFull, h.hz.x, ti + 1, R);
          h.hz.y = __shfl_sync(kFull, h.hz.y, ti + 1, R);
        }
      }
    }
    if (col < m) {
      o[0] = old[0] + (h.psi.x + h.psi.y);
      if (GRAD) {
        o[cstride] = old[1] + (h.hx.x + h.hx.y);
        o[2 * cstride] = old[2] + (h.hy.x + h.hy.y);
        o[3 * cstride] = old[3] + (h.hz.x + h.hz.y);
      }
    }
  }
}

// Per-warp shared memory: two column buffers (fills of kFC columns, staged
// twice: 2 kFC records) with their destinations, the own-leaf records and
// the upper-segment table of the current leaf.
constexpr int kSelf = 64;
template <typename T>
struct WarpSmem {
  static constexpr int kFC = pr<T>::kFC;
  typename pr<T>::Rec col[2][2 * kFC];
  int32_t dst[2][kFC];
  typename pr<T>::Rec self[kSelf];
  int2 seg[32];           // (source row - first column, dst - first column) of upper segment e
  int32_t incl[32];       // inclusive end column of segment e (0-size for non-upper entries)
};

template <typename T, bool GUARD, bool GRAD>
__global__ void __launch_bounds__(32 * kMW, (sizeof(T) == 4 ? KIFMM_MUT_MINB : KIFMM_MUT_MINB / 2) /
                                                (GRAD ? 2 : 1))
p2p_mutual_kernel(
    const T* __restrict__ tx, const T* __restrict__ ty, const T* __restrict__ tz,
    int64_t n_leaves, const typename pr<T>::Rec* __restrict__ src4, int64_t npts,
    const int32_t* __restrict__ near_off, const int4* __restrict__ near_pack,
    const int32_t* __restrict__ order, int64_t nrhs, int64_t pstride, T* __restrict__ P) {
  using O = pr<T>;
  using Rec = typename O::Rec;
  using P2 = typename O::P2;
  constexpr int kFC = O::kFC;
  __shared__ WarpSmem<T> sm_all[kMW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  WarpSmem<T>& sm = sm_all[w];
  // one leaf per warp, heaviest first (order: leaves by descending work)
  const int64_t slot = (int64_t)blockIdx.x * kMW + w;
  if (slot >= n_leaves) return;
  const int64_t a = order ? order[slot] : slot;
  // near entries of the first leaf: (start, count, dst, leaf); entry 0 is the
  // leaf itself, its dst field holds the leaf's slot base
  int4 ent = make_int4(0, 0, 0, -1);
  int nent = 0;
  {
    const int n0 = near_off[a];
    nent = near_off[a + 1] - n0;
    if (lane < nent) ent = near_pack[n0 + lane];
  }
  {
    const int t0 = __shfl_sync(kFull, ent.x, 0), tc = __shfl_sync(kFull, ent.y, 0);
    const int32_t own_base = __shfl_sync(kFull, ent.z, 0);
    // upper segments: exclusive prefix of their sizes over the entries
    const int ucnt = (lane > 0 && lane < nent && ent.w > a) ? ent.y : 0;
    int incl = ucnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    const int ncols = __shfl_sync(kFull, incl, 31);
    const int excl = incl - ucnt;
    __syncwarp();
    sm.seg[lane] = make_int2(ent.x - excl, ent.z - excl);
    sm.incl[lane] = incl;
    __syncwarp();
    for (int64_t r = 0; r < nrhs; ++r) {
      const Rec* srow = src4 + r * npts;
      constexpr int NC = GRAD ? 4 : 1;             // component planes per right-hand side
      T* Pr = P + r * NC * pstride;
      for (int tb = 0; tb < tc; tb += 32) {
        const int n = min(32, tc - tb);
        const int h = (n + 3) >> 2;                            // lanes per group: >= n / 4
        const int lr = h <= 1 ? 0 : 32 - __clz(h - 1);       // R = 2^lr
        const int R = 1 << lr;
        const int grp = lane >> lr, ti = lane & (R - 1), f = 32 >> lr;
        // four targets per lane: ti, ti + R, ti + 2R, ti + 3R (dead ones
        // repeat target 0 with charge 0)
        bool live[4];
        int64_t it[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          live[u] = ti + u * R < n;
          it[u] = t0 + tb + (live[u] ? ti + u * R : 0);
        }
        // stage one fill of columns [k kFC, ...) into buffer k & 1: each
        // column twice (2R-record chunks), padded to whole 32-column rounds
        auto stage = [&](int k) {
          Rec* cb = sm.col[k & 1];
          int32_t* db = sm.dst[k & 1];
          const int c0 = k * kFC, m = min(kFC, ncols - c0), mp = (m + 31) & ~31;
          for (int cc = lane; cc < mp; cc += 32) {
            const int e2 = ((cc >> lr) << (lr + 1)) + (cc & (R - 1));
            if (cc < m) {
              const int c = c0 + cc;
              int e = 0;
#pragma unroll
              for (int st = 16; st > 0; st >>= 1)
                if (sm.incl[e + st - 1] <= c) e += st;
              const int2 sg = sm.seg[e];
              cp_async_rec<T>(cb + e2, srow + sg.x + c);
              cp_async_rec<T>(cb + e2 + R, srow + sg.x + c);
              db[cc] = sg.y + c;
            } else {
              cb[e2] = pad_col<T>();
              cb[e2 + R] = pad_col<T>();
            }
          }
          cp_async_commit();
        };
        const int nfill = (ncols + kFC - 1) / kFC;
        // own leaf (first kSelf records) and the first fill in flight together
        const int ms = min(kSelf, tc);
        for (int k = lane; k < ms; k += 32) cp_async_rec<T>(sm.self + k, srow + t0 + k);
        cp_async_commit();
        if (nfill) stage(0);
        Quad<T> tq;
        tq.X0 = O::mk(tx[it[0]], tx[it[1]]);
        tq.Y0 = O::mk(ty[it[0]], ty[it[1]]);
        tq.Z0 = O::mk(tz[it[0]], tz[it[1]]);
        tq.X1 = O::mk(tx[it[2]], tx[it[3]]);
        tq.Y1 = O::mk(ty[it[2]], ty[it[3]]);
        tq.Z1 = O::mk(tz[it[2]], tz[it[3]]);
        const P2 QA0 = O::mk(live[0] ? srow[it[0]].w : T(0), live[1] ? srow[it[1]].w : T(0));
        const P2 QA1 = O::mk(live[2] ? srow[it[2]].w : T(0), live[3] ? srow[it[3]].w : T(0));
        Rows<T> acc;
        acc.phi0 = acc.phi1 = acc.g0x = acc.g0y = acc.g0z = acc.g1x = acc.g1y = acc.g1z =
            O::mk(T(0), T(0));
        // ---- own block (direct, guarded)
        if (nfill) cp_async_wait<1>();
        else cp_async_wait<0>();
        __syncwarp();
        self_sum<T, GRAD>(sm.self, ms, grp, f, tq, acc);
        for (int j0 = kSelf; j0 < tc; j0 += kSelf) {           // large leaves: more pieces
          const int m = min(kSelf, tc - j0);
          __syncwarp();
          for (int k = lane; k < m; k += 32) cp_async_rec<T>(sm.self + k, srow + t0 + j0 + k);
          cp_async_commit();
          cp_async_wait<0>();                                  // (also completes fill 0)
          __syncwarp();
          self_sum<T, GRAD>(sm.self, m, grp, f, tq, acc);
        }
        // ---- upper blocks: double-buffered fills
        const bool rmw = tb > 0;
        for (int k = 0; k < nfill; ++k) {
          if (k + 1 < nfill) {
            stage(k + 1);
            cp_async_wait<1>();
          } else {
            cp_async_wait<0>();
          }
          __syncwarp();
          const Rec* cb = sm.col[k & 1];
          const int32_t* db = sm.dst[k & 1];
          const int m = min(kFC, ncols - k * kFC);
          switch (lr) {
            case 0: mutual_rounds<T, 1, GUARD, GRAD>(cb, db, m, grp, ti, tq, QA0, QA1, acc, Pr, pstride, rmw); break;
            case 1: mutual_rounds<T, 2, GUARD, GRAD>(cb, db, m, grp, ti, tq, QA0, QA1, acc, Pr, pstride, rmw); break;
            case 2: mutual_rounds<T, 4, GUARD, GRAD>(cb, db, m, grp, ti, tq, QA0, QA1, acc, Pr, pstride, rmw); break;
            default: mutual_rounds<T, 8, GUARD, GRAD>(cb, db, m, grp, ti, tq, QA0, QA1, acc, Pr, pstride, rmw); break;
          }
          __syncwarp();
        }
        // ---- row sums of the pass: combine the f groups, slot 0 (the
        // gradient rows with their sign: grad phi = -G)
        T ph[4 * NC] = {acc.phi0.x, acc.phi0.y, acc.phi1.x, acc.phi1.y};
        if (GRAD) {
          const T gv[12] = {acc.g0x.x, acc.g0x.y, acc.g1x.x, acc.g1x.y, acc.g0y.x, acc.g0y.y,
                            acc.g1y.x, acc.g1y.y, acc.g0z.x, acc.g0z.y, acc.g1z.x, acc.g1z.y};
#pragma unroll
          for (int u = 0; u < 12; ++u) ph[(GRAD ? 4 : 0) + u] = -gv[u];
        }
        for (int off = R; off < 32; off <<= 1) {
#pragma unroll
          for (int u = 0; u < 4 * NC; ++u) ph[u] += __shfl_xor_sync(kFull, ph[u], off);
        }
        if (grp == 0) {
#pragma unroll
          for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (live[u]) Pr[c * pstride + own_base + tb + ti + u * R] = ph[4 * c + u];
        }
        __syncwarp();
      }
    }
  }
}

// Near-field totals: out[perm[i]] = (1/4pi) sum_s P[slot s of i], slots in
// order, for every target of leaf b (one warp per leaf, a lane per target);
// runs right after the mutual pass, concurrently with the far field, and the
// final L2P pass accumulates onto it (kifmm_leaf_pass_f32, parts = 1 | 4).
constexpr int kRW = 8;
template <typename T, bool GRAD>
__global__ void __launch_bounds__(32 * kRW, 4) mutual_reduce_kernel(
    const int32_t* __restrict__ tstart, const int32_t* __restrict__ tcount, int64_t n_tleaves,
    int64_t nrhs, const int64_t* __restrict__ perm, const int32_t* __restrict__ base,
    const int32_t* __restrict__ nlow, int64_t pstride, const T* __restrict__ P,
    T* __restrict__ out, T* __restrict__ grad) {
  constexpr int NC = GRAD ? 4 : 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * kRW + w;
  if (b >= n_tleaves) return;
  const int64_t t0 = tstart[b];
  const int tc = tcount[b];
  const int slots = 1 + nlow[b];
  const int32_t pb0 = base[b];
  const T c = real_traits<T>::inv4pi();
  for (int t = lane; t < tc; t += 32) {
    const int64_t o = perm ? perm[t0 + t] : t0 + t;
    for (int64_t r = 0; r < nrhs; ++r) {
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        const T* Pr = P + (r * NC + cc) * pstride + pb0 + t;
        T acc = T(0);
        // slots in order, eight loads in flight at a time
        for (int s0 = 0; s0 < slots; s0 += 8) {
          T v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = s0 + u < slots ? __ldg(Pr + (s0 + u) * tc) : T(0);
#pragma unroll
          for (int u = 0; u < 8; ++u) acc += v[u];
        }
        if (cc == 0) out[o * nrhs + r] = acc * c;
        else grad[(o * nrhs + r) * 3 + (cc - 1)] = acc * c;
      }
    }
  }
}

template <typename T, bool GRAD>
int p2p_mutual(const T* tx, const T* ty, const T* tz, int64_t n_leaves, const T* src4, int64_t npts,
               const int32_t* near_off, const int32_t* near_pack, const int32_t* order,
               int64_t nrhs, int64_t pstride, int guard, T* P, void* stream) {
  if (n_leaves < 0 || npts < 0 || nrhs < 1 || pstride < npts) return KIFMM_EARG;
  if (n_leaves == 0) return 0;
  const auto* s4 = reinterpret_cast<const typename pr<T>::Rec*>(src4);
  const auto* pk = reinterpret_cast<const int4*>(near_pack);
  const unsigned grid = ceil_div(n_leaves, kMW);
  if (guard)
    p2p_mutual_kernel<T, true, GRAD><<<grid, 32 * kMW, 0, (cudaStream_t)stream>>>(
        tx, ty, tz, n_leaves, s4, npts, near_off, pk, order, nrhs, pstride, P);
  else
    p2p_mutual_kernel<T, false, GRAD><<<grid, 32 * kMW, 0, (cudaStream_t)stream>>>(
        tx, ty, tz, n_leaves, s4, npts, near_off, pk, order, nrhs, pstride, P);
  return launch_status();
}

template <typename T, bool GRAD>
int mutual_reduce(const int32_t* ts, const int32_t* tc, int64_t ntl, int64_t nrhs,
                  const int64_t* perm, const int32_t* base, const int32_t* nlow, int64_t pstride,
                  const T* P, T* out, T* grad, void* stream) {
  if (ntl < 0 || nrhs < 1 || (GRAD && !grad)) return KIFMM_EARG;
  if (ntl == 0) return 0;
  mutual_reduce_kernel<T, GRAD><<<ceil_div(ntl, kRW), 32 * kRW, 0, (cudaStream_t)stream>>>(
      ts, tc, ntl, nrhs, perm, base, nlow, pstride, P, out, grad);
  return launch_status();
}

}  // namespace

extern "C" {

// Mutual near field into the partial-sum slots P (layout above); sources ==
// targets, tree order.  src4: (nrhs, npts) records (x, y, z, q); near_dst[e]
// = base_B + slot * n_B for an upper entry e of leaf A's near list (B > A),
// unused otherwise; P: nrhs planes of pstride elements.
int kifmm_p2p_mutual_f32(const float* tx, const float* ty, const float* tz, int64_t n_leaves,
                         const float* src4, int64_t npts, const int32_t* near_off,
                         const int32_t* near_pack, const int32_t* order, int64_t nrhs,
                         int64_t pstride, int guard, float* P, void* stream) {
  return p2p_mutual<float, false>(tx, ty, tz, n_leaves, src4, npts, near_off, near_pack, order,
                                  nrhs, pstride, guard, P, stream);
}
int kifmm_p2p_mutual_f64(const double* tx, const double* ty, const double* tz, int64_t n_leaves,
                         const double* src4, int64_t npts, const int32_t* near_off,
                         const int32_t* near_pack, const int32_t* order, int64_t nrhs,
                         int64_t pstride, int guard, double* P, void* stream) {
  return p2p_mutual<double, false>(tx, ty, tz, n_leaves, src4, npts, near_off, near_pack, order,
                                   nrhs, pstride, guard, P, stream);
}

// out[perm[i]] = (1/4pi) sum of i's near-field slots (slot order).
int kifmm_p2p_mutual_reduce_f32(const int32_t* ts, const int32_t* tc, int64_t ntl, int64_t nrhs,
                                const int64_t* perm, const int32_t* base, const int32_t* nlow,
                                int64_t pstride, const float* P, float* out, void* stream) {
  return mutual_reduce<float, false>(ts, tc, ntl, nrhs, perm, base, nlow, pstride, P, out, nullptr,
                                     stream);
}
int kifmm_p2p_mutual_reduce_f64(const int32_t* ts, const int32_t* tc, int64_t ntl, int64_t nrhs,
                                const int64_t* perm, const int32_t* base, const int32_t* nlow,
                                int64_t pstride, const double* P, double* out, void* stream) {
  return mutual_reduce<double, false>(ts, tc, ntl, nrhs, perm, base, nlow, pstride, P, out, nullptr,
                                      stream);
}


// Potential + gradient (BASELINE config 3; the reference is potential-only):
// P holds four component planes per right-hand side (potential, then d/dx,
// d/dy, d/dz: P[(r*4 + c)*pstride + slot]), grad is (target, rhs, 3).
int kifmm_p2p_mutual_grad_f32(const float* tx, const float* ty, const float* tz, int64_t n_leaves,
                              const float* src4, int64_t npts, const int32_t* near_off,
                              const int32_t* near_pack, const int32_t* order, int64_t nrhs,
                              int64_t pstride, int guard, float* P, void* stream) {
  return p2p_mutual<float, true>(tx, ty, tz, n_leaves, src4, npts, near_off, near_pack, order,
                                 nrhs, pstride, guard, P, stream);
}
int kifmm_p2p_mutual_grad_f64(const double* tx, const double* ty, const double* tz,
                              int64_t n_leaves, const double* src4, int64_t npts,
                              const int32_t* near_off, const int32_t* near_pack,
                              const int32_t* order, int64_t nrhs, int64_t pstride, int guard,
                              double* P, void* stream) {
  return p2p_mutual<double, true>(tx, ty, tz, n_leaves, src4, npts, near_off, near_pack, order,
                                  nrhs, pstride, guard, P, stream);
}
int kifmm_p2p_mutual_reduce_grad_f32(const int32_t* ts, const int32_t* tc, int64_t ntl,
                                     int64_t nrhs, const int64_t* perm, const int32_t* base,
                                     const int32_t* nlow, int64_t pstride, const float* P,
                                     float* out, float* grad, void* stream) {
  return mutual_reduce<float, true>(ts, tc, ntl, nrhs, perm, base, nlow, pstride, P, out, grad,
                                    stream);
}
int kifmm_p2p_mutual_reduce_grad_f64(const int32_t* ts, const int32_t* tc, int64_t ntl,
                                     int64_t nrhs, const int64_t* perm, const int32_t* base,
                                     const int32_t* nlow, int64_t pstride, const double* P,
                                     double* out, double* grad, void* stream) {
  return mutual_reduce<double, true>(ts, tc, ntl, nrhs, perm, base, nlow, pstride, P, out, grad,
                                     stream);
}

}  // extern "C"
