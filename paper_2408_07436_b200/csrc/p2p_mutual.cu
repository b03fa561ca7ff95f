// Mutual (symmetric) near field for sources == targets, float32, potential.
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

__device__ __forceinline__ float4 pad_col() {
  // far-away, chargeless: r2 = inf -> rsqrt = 0, no contribution either way
  return make_float4(__int_as_float(0x7f800000), __int_as_float(0x7f800000),
                     __int_as_float(0x7f800000), 0.f);
}

// Row-only sum over staged records [0, m) for the lane's four targets (two
// packed pairs: X0 = targets (0, 1), X1 = (2, 3)), sources j = start,
// start + stride, ...; every record may coincide with a target (the leaf's
// own block): r2 = 0 contributes 0.
struct Quad {
  float2 X0, Y0, Z0, X1, Y1, Z1;
};
__device__ __forceinline__ float2 inv_r2(float2 X, float2 Y, float2 Z, const float4& s) {
  const float2 dx = __fadd2_rn(X, make_float2(-s.x, -s.x));
  const float2 dy = __fadd2_rn(Y, make_float2(-s.y, -s.y));
  const float2 dz = __fadd2_rn(Z, make_float2(-s.z, -s.z));
  return __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
}
template <bool GUARD>
__device__ __forceinline__ float2 rsq2f(float2 r2) {
  float w0 = real_traits<float>::rsq(r2.x), w1 = real_traits<float>::rsq(r2.y);
  if (GUARD) {
    w0 = r2.x > 0.f ? w0 : 0.f;
    w1 = r2.y > 0.f ? w1 : 0.f;
  }
  return make_float2(w0, w1);
}
__device__ __forceinline__ void self_sum(const float4* buf, int m, int start, int stride,
                                         const Quad& t, float2& acc0, float2& acc1) {
  for (int j = start; j < m; j += stride) {
    const float4 s = buf[j];
    const float2 q = make_float2(s.w, s.w);
    acc0 = __ffma2_rn(rsq2f<true>(inv_r2(t.X0, t.Y0, t.Z0, s)), q, acc0);
    acc1 = __ffma2_rn(rsq2f<true>(inv_r2(t.X1, t.Y1, t.Z1, s)), q, acc1);
  }
}

// Rounds of 32 staged columns (f chunks of R); group grp takes chunk
// round * f + grp.  Chunk k occupies buf[2Rk, 2Rk + 2R) (the chunk twice).
// Per step a lane meets one column with its four targets: one 16-byte
// shared load and two shuffles feed four interactions.
template <int R, bool GUARD>
__device__ __forceinline__ void mutual_rounds(const float4* buf, const int32_t* dst, int m,
                                              int grp, int ti, const Quad& t, float2 QA0,
                                              float2 QA1, float2& phi0, float2& phi1,
                                              float* __restrict__ Pr, bool rmw) {
  for (int c0 = 0; c0 < m; c0 += 32) {
    const int k = c0 / R + grp;                    // R is a compile-time power of two
    const float4* p = buf + 2 * R * k + ti;
    const int col = k * R + ti;
    // a later target pass of the same leaf adds to the column sums of the
    // earlier ones: fetch them before the chain of steps
    float* o = Pr + (col < m ? dst[col] : 0);
    const float old = (rmw && col < m) ? __ldcg(o) : 0.f;
    float2 psi = make_float2(0.f, 0.f);
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const float4 c = p[s];
      const float2 w0 = rsq2f<GUARD>(inv_r2(t.X0, t.Y0, t.Z0, c));
      const float2 w1 = rsq2f<GUARD>(inv_r2(t.X1, t.Y1, t.Z1, c));
      const float2 q = make_float2(c.w, c.w);
      phi0 = __ffma2_rn(w0, q, phi0);
      phi1 = __ffma2_rn(w1, q, phi1);
      psi = __ffma2_rn(w1, QA1, __ffma2_rn(w0, QA0, psi));
      if (R > 1) {
        psi.x = __shfl_sync(kFull, psi.x, ti + 1, R);
        psi.y = __shfl_sync(kFull, psi.y, ti + 1, R);
      }
    }
    if (col < m) *o = old + (psi.x + psi.y);
  }
}

// Per-warp shared memory: two column buffers (fills of kFC columns, staged
// twice: 2 kFC records) with their destinations, the own-leaf records and
// the upper-segment table of the current leaf.
constexpr int kFC = 128;
constexpr int kSelf = 64;
struct WarpSmem {
  float4 col[2][2 * kFC];
  int32_t dst[2][kFC];
  float4 self[kSelf];
  int2 seg[32];           // (source row - first column, dst - first column) of upper segment e
  int32_t incl[32];       // inclusive end column of segment e (0-size for non-upper entries)
};

template <bool GUARD>
__global__ void __launch_bounds__(32 * kMW, KIFMM_MUT_MINB) p2p_mutual_kernel(
    const float* __restrict__ tx, const float* __restrict__ ty, const float* __restrict__ tz,
    int64_t n_leaves, const float4* __restrict__ src4, int64_t npts,
    const int32_t* __restrict__ near_off, const int4* __restrict__ near_pack,
    const int32_t* __restrict__ order, int64_t nrhs, int64_t pstride, float* __restrict__ P) {
  __shared__ WarpSmem sm_all[kMW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  WarpSmem& sm = sm_all[w];
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
      const float4* srow = src4 + r * npts;
      float* Pr = P + r * pstride;
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
          float4* cb = sm.col[k & 1];
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
              cp_async16(cb + e2, srow + sg.x + c, true);
              cp_async16(cb + e2 + R, srow + sg.x + c, true);
              db[cc] = sg.y + c;
            } else {
              cb[e2] = pad_col();
              cb[e2 + R] = pad_col();
            }
          }
          cp_async_commit();
        };
        const int nfill = (ncols + kFC - 1) / kFC;
        // own leaf (first kSelf records) and the first fill in flight together
        const int ms = min(kSelf, tc);
        for (int k = lane; k < ms; k += 32) cp_async16(sm.self + k, srow + t0 + k, true);
        cp_async_commit();
        if (nfill) stage(0);
        Quad tq;
        tq.X0 = make_float2(tx[it[0]], tx[it[1]]);
        tq.Y0 = make_float2(ty[it[0]], ty[it[1]]);
        tq.Z0 = make_float2(tz[it[0]], tz[it[1]]);
        tq.X1 = make_float2(tx[it[2]], tx[it[3]]);
        tq.Y1 = make_float2(ty[it[2]], ty[it[3]]);
        tq.Z1 = make_float2(tz[it[2]], tz[it[3]]);
        const float2 QA0 = make_float2(live[0] ? srow[it[0]].w : 0.f, live[1] ? srow[it[1]].w : 0.f);
        const float2 QA1 = make_float2(live[2] ? srow[it[2]].w : 0.f, live[3] ? srow[it[3]].w : 0.f);
        float2 phi0 = make_float2(0.f, 0.f), phi1 = make_float2(0.f, 0.f);
        // ---- own block (direct, guarded)
        if (nfill) cp_async_wait<1>();
        else cp_async_wait<0>();
        __syncwarp();
        self_sum(sm.self, ms, grp, f, tq, phi0, phi1);
        for (int j0 = kSelf; j0 < tc; j0 += kSelf) {           // large leaves: more pieces
          const int m = min(kSelf, tc - j0);
          __syncwarp();
          for (int k = lane; k < m; k += 32) cp_async16(sm.self + k, srow + t0 + j0 + k, true);
          cp_async_commit();
          cp_async_wait<0>();                                  // (also completes fill 0)
          __syncwarp();
          self_sum(sm.self, m, grp, f, tq, phi0, phi1);
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
          const float4* cb = sm.col[k & 1];
          const int32_t* db = sm.dst[k & 1];
          const int m = min(kFC, ncols - k * kFC);
          switch (lr) {
            case 0: mutual_rounds<1, GUARD>(cb, db, m, grp, ti, tq, QA0, QA1, phi0, phi1, Pr, rmw); break;
            case 1: mutual_rounds<2, GUARD>(cb, db, m, grp, ti, tq, QA0, QA1, phi0, phi1, Pr, rmw); break;
            case 2: mutual_rounds<4, GUARD>(cb, db, m, grp, ti, tq, QA0, QA1, phi0, phi1, Pr, rmw); break;
            default: mutual_rounds<8, GUARD>(cb, db, m, grp, ti, tq, QA0, QA1, phi0, phi1, Pr, rmw); break;
          }
          __syncwarp();
        }
        // ---- row sums of the pass: combine the f groups, slot 0
        float ph[4] = {phi0.x, phi0.y, phi1.x, phi1.y};
        for (int off = R; off < 32; off <<= 1) {
#pragma unroll
          for (int u = 0; u < 4; ++u) ph[u] += __shfl_xor_sync(kFull, ph[u], off);
        }
        if (grp == 0) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (live[u]) Pr[own_base + tb + ti + u * R] = ph[u];
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
__global__ void __launch_bounds__(32 * kRW, 4) mutual_reduce_kernel(
    const int32_t* __restrict__ tstart, const int32_t* __restrict__ tcount, int64_t n_tleaves,
    int64_t nrhs, const int64_t* __restrict__ perm, const int32_t* __restrict__ base,
    const int32_t* __restrict__ nlow, int64_t pstride, const float* __restrict__ P,
    float* __restrict__ out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * kRW + w;
  if (b >= n_tleaves) return;
  const int64_t t0 = tstart[b];
  const int tc = tcount[b];
  const int slots = 1 + nlow[b];
  const int32_t pb0 = base[b];
  const float c = real_traits<float>::inv4pi();
  for (int t = lane; t < tc; t += 32) {
    const int64_t o = perm ? perm[t0 + t] : t0 + t;
    for (int64_t r = 0; r < nrhs; ++r) {
      const float* Pr = P + r * pstride + pb0 + t;
      float acc = 0.f;
      // slots in order, eight loads in flight at a time
      for (int s0 = 0; s0 < slots; s0 += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = s0 + u < slots ? __ldg(Pr + (s0 + u) * tc) : 0.f;
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
      }
      out[o * nrhs + r] = acc * c;
    }
  }
}

}  // namespace

extern "C" {

// Mutual near field into the partial-sum slots P (layout above); sources ==
// targets, tree order.  src4: (nrhs, npts) records (x, y, z, q); near_dst[e]
// = base_B + slot * n_B for an upper entry e of leaf A's near list (B > A),
// unused otherwise; P: nrhs planes of pstride floats.
int kifmm_p2p_mutual_f32(const float* tx, const float* ty, const float* tz, int64_t n_leaves,
                         const float* src4, int64_t npts, const int32_t* near_off,
                         const int32_t* near_pack, const int32_t* order, int64_t nrhs,
                         int64_t pstride, int guard, float* P, void* stream) {
  if (n_leaves < 0 || npts < 0 || nrhs < 1 || pstride < npts) return KIFMM_EARG;
  if (n_leaves == 0) return 0;
  const auto* s4 = reinterpret_cast<const float4*>(src4);
  const auto* pk = reinterpret_cast<const int4*>(near_pack);
  const unsigned grid = ceil_div(n_leaves, kMW);
  if (guard)
    p2p_mutual_kernel<true><<<grid, 32 * kMW, 0, (cudaStream_t)stream>>>(
        tx, ty, tz, n_leaves, s4, npts, near_off, pk, order, nrhs, pstride, P);
  else
    p2p_mutual_kernel<false><<<grid, 32 * kMW, 0, (cudaStream_t)stream>>>(
        tx, ty, tz, n_leaves, s4, npts, near_off, pk, order, nrhs, pstride, P);
  return launch_status();
}

// out[perm[i]] = (1/4pi) sum of i's near-field slots (slot order).
int kifmm_p2p_mutual_reduce_f32(const int32_t* ts, const int32_t* tc, int64_t ntl, int64_t nrhs,
                                const int64_t* perm, const int32_t* base, const int32_t* nlow,
                                int64_t pstride, const float* P, float* out, void* stream) {
  if (ntl < 0 || nrhs < 1) return KIFMM_EARG;
  if (ntl == 0) return 0;
  mutual_reduce_kernel<<<ceil_div(ntl, kRW), 32 * kRW, 0, (cudaStream_t)stream>>>(
      ts, tc, ntl, nrhs, perm, base, nlow, pstride, P, out);
  return launch_status();
}

}  // extern "C"
