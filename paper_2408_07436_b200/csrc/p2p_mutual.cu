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
// at P[base_B + s n_B + t]; l2p_mutual_kernel adds the slots of each target
// in slot order to its L2P far field and un-permutes (engine.py:377-404).
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

constexpr int kMW = 4;              // warps per CTA (one target leaf per warp)
constexpr int kMCols = 256;         // upper columns staged per fill (x2 entries: the chunk twice)
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float4 pad_col() {
  // far-away, chargeless: r2 = inf -> rsqrt = 0, no contribution either way
  return make_float4(__int_as_float(0x7f800000), __int_as_float(0x7f800000),
                     __int_as_float(0x7f800000), 0.f);
}

// Row-only sum over staged records [0, m) for the lane's two packed targets,
// sources j = start, start + stride, ...; every record may coincide with a
// target (the leaf's own block): r2 = 0 contributes 0.
__device__ __forceinline__ void self_sum(const float4* buf, int m, int start, int stride,
                                         float2 X, float2 Y, float2 Z, float2& acc) {
  float2 acc2 = make_float2(0.f, 0.f);
  auto body = [&](int j, float2& a_) {
    const float4 s = buf[j];
    const float2 dx = __fadd2_rn(X, make_float2(-s.x, -s.x));
    const float2 dy = __fadd2_rn(Y, make_float2(-s.y, -s.y));
    const float2 dz = __fadd2_rn(Z, make_float2(-s.z, -s.z));
    const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
    float w0 = real_traits<float>::rsq(r2.x), w1 = real_traits<float>::rsq(r2.y);
    w0 = r2.x > 0.f ? w0 : 0.f;
    w1 = r2.y > 0.f ? w1 : 0.f;
    a_ = __ffma2_rn(make_float2(w0, w1), make_float2(s.w, s.w), a_);
  };
  int j = start;
  for (; j + stride < m; j += 2 * stride) {
    body(j, acc);
    body(j + stride, acc2);
  }
  if (j < m) body(j, acc);
  acc = __fadd2_rn(acc, acc2);
}

// Rounds of 32 staged columns (f chunks of R); group grp takes chunk
// round * f + grp.  Chunk k occupies buf[2Rk, 2Rk + 2R) (the chunk twice).
template <int R, bool GUARD>
__device__ __forceinline__ void mutual_rounds(const float4* buf, const int32_t* dst, int m,
                                              int grp, int ti, float2 X, float2 Y, float2 Z,
                                              float2 QA, float2& phi, float* __restrict__ Pr,
                                              bool rmw) {
  for (int c0 = 0; c0 < m; c0 += 32) {
    const int k = c0 / R + grp;
    const float4* p = buf + 2 * R * k + ti;
    float2 psi = make_float2(0.f, 0.f);
    float2 acc2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int s = 0; s < R; ++s) {
      const float4 c = p[s];
      const float2 dx = __fadd2_rn(X, make_float2(-c.x, -c.x));
      const float2 dy = __fadd2_rn(Y, make_float2(-c.y, -c.y));
      const float2 dz = __fadd2_rn(Z, make_float2(-c.z, -c.z));
      const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
      float w0 = real_traits<float>::rsq(r2.x), w1 = real_traits<float>::rsq(r2.y);
      if (GUARD) {
        w0 = r2.x > 0.f ? w0 : 0.f;
        w1 = r2.y > 0.f ? w1 : 0.f;
      }
      const float2 w = make_float2(w0, w1);
      if (s & 1) acc2 = __ffma2_rn(w, make_float2(c.w, c.w), acc2);
      else phi = __ffma2_rn(w, make_float2(c.w, c.w), phi);
      psi = __ffma2_rn(w, QA, psi);
      if (R > 1) {
        psi.x = __shfl_sync(kFull, psi.x, ti + 1, R);
        psi.y = __shfl_sync(kFull, psi.y, ti + 1, R);
      }
    }
    phi = __fadd2_rn(phi, acc2);
    const int col = k * R + ti;
    if (col < m) {
      float* o = Pr + dst[col];
      const float v = psi.x + psi.y;
      *o = rmw ? __ldcg(o) + v : v;
    }
  }
}

template <bool GUARD>
__global__ void __launch_bounds__(32 * kMW) p2p_mutual_kernel(
    const float* __restrict__ tx, const float* __restrict__ ty, const float* __restrict__ tz,
    const int32_t* __restrict__ lstart, const int32_t* __restrict__ lcount, int64_t n_leaves,
    const float4* __restrict__ src4, int64_t npts, const int32_t* __restrict__ near_off,
    const int32_t* __restrict__ near_leaf, const int32_t* __restrict__ near_dst,
    const int32_t* __restrict__ base, int64_t nrhs, int64_t pstride, float* __restrict__ P) {
  __shared__ __align__(16) float4 sbuf[kMW][2 * kMCols];
  __shared__ int32_t sdst[kMW][kMCols];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4* buf = sbuf[w];
  int32_t* dsts = sdst[w];
  const int64_t a = (int64_t)blockIdx.x * kMW + w;
  if (a >= n_leaves) return;
  const int64_t t0 = lstart[a];
  const int tc = lcount[a];
  const int n0 = near_off[a], n1 = near_off[a + 1];
  // near entries by lane (<= 27): upper neighbours are the entries whose leaf
  // row is above a (own leaf first, then neighbours ascending)
  int seg_start = 0, seg_cnt = 0, seg_dst = 0;
  bool upper = false;
  if (lane < n1 - n0) {
    const int sl = near_leaf[n0 + lane];
    seg_start = lstart[sl];
    seg_cnt = lcount[sl];
    seg_dst = near_dst[n0 + lane];
    upper = sl > a;
  }
  const unsigned umask = __ballot_sync(kFull, upper);
  const int32_t own_base = base[a];
  for (int64_t r = 0; r < nrhs; ++r) {
    const float4* srow = src4 + r * npts;
    float* Pr = P + r * pstride;
    for (int tb = 0; tb < tc; tb += 32) {
      const int n = min(32, tc - tb);
      const int h = (n + 1) >> 1;
      const int R = h <= 1 ? 1 : 1 << (32 - __clz(h - 1));
      const int f = 32 / R, grp = lane / R, ti = lane % R;
      const bool live0 = ti < n, live1 = ti + R < n;
      const int64_t ia = t0 + tb + (live0 ? ti : 0), ib = t0 + tb + (live1 ? ti + R : 0);
      const float2 X = make_float2(tx[ia], tx[ib]), Y = make_float2(ty[ia], ty[ib]),
                   Z = make_float2(tz[ia], tz[ib]);
      const float2 QA = make_float2(live0 ? srow[ia].w : 0.f, live1 ? srow[ib].w : 0.f);
      float2 phi = make_float2(0.f, 0.f);
      // ---- own block (direct, guarded), in pieces of 2 kMCols records
      for (int j0 = 0; j0 < tc; j0 += 2 * kMCols) {
        const int m = min(2 * kMCols, tc - j0);
        __syncwarp();
        for (int k = lane; k < m; k += 32) cp_async16(buf + k, srow + t0 + j0 + k, true);
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        self_sum(buf, m, grp, f, X, Y, Z, phi);
      }
      // ---- upper blocks: columns of all upper neighbours, kMCols per fill
      int fill = 0;
      auto process = [&](int m) {
        // pad to whole rounds of 32 columns
        const int mp = (m + 31) & ~31;
        for (int c = m + lane; c < mp; c += 32) {
          const int k = c / R, pos = c % R;
          buf[2 * R * k + pos] = pad_col();
          buf[2 * R * k + R + pos] = pad_col();
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        const bool rmw = tb > 0;
        switch (R) {
          case 1: mutual_rounds<1, GUARD>(buf, dsts, m, grp, ti, X, Y, Z, QA, phi, Pr, rmw); break;
          case 2: mutual_rounds<2, GUARD>(buf, dsts, m, grp, ti, X, Y, Z, QA, phi, Pr, rmw); break;
          case 4: mutual_rounds<4, GUARD>(buf, dsts, m, grp, ti, X, Y, Z, QA, phi, Pr, rmw); break;
          case 8: mutual_rounds<8, GUARD>(buf, dsts, m, grp, ti, X, Y, Z, QA, phi, Pr, rmw); break;
          default: mutual_rounds<16, GUARD>(buf, dsts, m, grp, ti, X, Y, Z, QA, phi, Pr, rmw); break;
        }
        __syncwarp();
      };
      __syncwarp();
      unsigned um = umask;
      while (um) {
        const int nn = __ffs(um) - 1;
        um &= um - 1;
        const int64_t j0 = __shfl_sync(kFull, seg_start, nn);
        const int jc = __shfl_sync(kFull, seg_cnt, nn);
        const int32_t d0 = __shfl_sync(kFull, seg_dst, nn);
        for (int jb = 0; jb < jc;) {
          if (fill == kMCols) {
            process(fill);
            fill = 0;
          }
          const int m = min(jc - jb, kMCols - fill);
          for (int k = lane; k < m; k += 32) {
            const int c = fill + k, ck = c / R, pos = c % R;
            cp_async16(buf + 2 * R * ck + pos, srow + j0 + jb + k, true);
            cp_async16(buf + 2 * R * ck + R + pos, srow + j0 + jb + k, true);
            dsts[c] = d0 + jb + k;
          }
          fill += m;
          jb += m;
        }
      }
      if (fill) process(fill);
      // ---- row sums of the pass: combine the f groups, slot 0
      float pa = phi.x, pb = phi.y;
      for (int off = R; off < 32; off <<= 1) {
        pa += __shfl_xor_sync(kFull, pa, off);
        pb += __shfl_xor_sync(kFull, pb, off);
      }
      if (grp == 0) {
        if (live0) Pr[own_base + tb + ti] = pa;
        if (live1) Pr[own_base + tb + ti + R] = pb;
      }
      __syncwarp();
    }
  }
}

// Final pass: L2P (downward equivalent surface -> targets) + the near-field
// slots of each target in slot order, un-permuted to caller order.
constexpr int kLW = 8;
__global__ void __launch_bounds__(32 * kLW) l2p_mutual_kernel(
    const float* __restrict__ tx, const float* __restrict__ ty, const float* __restrict__ tz,
    const int32_t* __restrict__ tstart, const int32_t* __restrict__ tcount, int64_t n_tleaves,
    const double* __restrict__ centers, const double* __restrict__ ebase, int ne,
    const float* __restrict__ local, int64_t nrhs, const int64_t* __restrict__ perm,
    const int32_t* __restrict__ base, const int32_t* __restrict__ nlow, int64_t pstride,
    const float* __restrict__ P, float* __restrict__ out) {
  extern __shared__ __align__(16) float4 l2pm_buf[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4* buf = l2pm_buf + w * ne;
  const int64_t b = (int64_t)blockIdx.x * kLW + w;
  if (b >= n_tleaves) return;
  const int64_t t0 = tstart[b];
  const int tc = tcount[b];
  const int slots = 1 + nlow[b];
  const int32_t pb0 = base[b];
  const double cx = centers[b * 3], cy = centers[b * 3 + 1], cz = centers[b * 3 + 2];
  for (int tb = 0; tb < tc; tb += 32) {
    const int n = min(32, tc - tb);
    const int h = (n + 1) >> 1;
    const int R = h <= 1 ? 1 : 1 << (32 - __clz(h - 1));
    const int f = 32 / R, sub = lane / R;
    const int ti = lane % R;
    const bool live0 = ti < n, live1 = ti + R < n;
    const int64_t ia = t0 + tb + (live0 ? ti : 0), ib = t0 + tb + (live1 ? ti + R : 0);
    const float2 X = make_float2(tx[ia], tx[ib]), Y = make_float2(ty[ia], ty[ib]),
                 Z = make_float2(tz[ia], tz[ib]);
    const int64_t oa = perm ? perm[ia] : ia, ob = perm ? perm[ib] : ib;
    for (int64_t r = 0; r < nrhs; ++r) {
      const float* loc = local + (b * nrhs + r) * ne;
      // near field: the target's slots, in slot order (issued before the
      // interaction loop; independent loads)
      float na = 0.f, nb = 0.f;
      if (sub == 0) {
        const float* Pr = P + r * pstride + pb0 + tb + ti;
        for (int s = 0; s < slots; ++s) {
          if (live0) na += __ldg(Pr + (int64_t)s * tc);
          if (live1) nb += __ldg(Pr + (int64_t)s * tc + R);
        }
      }
      __syncwarp();
      for (int k = lane; k < ne; k += 32)
        buf[k] = make_float4(real_traits<float>::from_d(exact_add(cx, ebase[k * 3])),
                             real_traits<float>::from_d(exact_add(cy, ebase[k * 3 + 1])),
                             real_traits<float>::from_d(exact_add(cz, ebase[k * 3 + 2])), loc[k]);
      __syncwarp();
      float2 acc = make_float2(0.f, 0.f), acc2 = make_float2(0.f, 0.f);
      int k = sub;
      for (; k + f < ne; k += 2 * f) {
        const float4 s = buf[k], s2 = buf[k + f];
        float2 dx = __fadd2_rn(X, make_float2(-s.x, -s.x));
        float2 dy = __fadd2_rn(Y, make_float2(-s.y, -s.y));
        float2 dz = __fadd2_rn(Z, make_float2(-s.z, -s.z));
        float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
        acc = __ffma2_rn(make_float2(real_traits<float>::rsq(r2.x), real_traits<float>::rsq(r2.y)),
                         make_float2(s.w, s.w), acc);
        dx = __fadd2_rn(X, make_float2(-s2.x, -s2.x));
        dy = __fadd2_rn(Y, make_float2(-s2.y, -s2.y));
        dz = __fadd2_rn(Z, make_float2(-s2.z, -s2.z));
        r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
        acc2 = __ffma2_rn(make_float2(real_traits<float>::rsq(r2.x), real_traits<float>::rsq(r2.y)),
                          make_float2(s2.w, s2.w), acc2);
      }
      if (k < ne) {
        const float4 s = buf[k];
        const float2 dx = __fadd2_rn(X, make_float2(-s.x, -s.x));
        const float2 dy = __fadd2_rn(Y, make_float2(-s.y, -s.y));
        const float2 dz = __fadd2_rn(Z, make_float2(-s.z, -s.z));
        const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
        acc = __ffma2_rn(make_float2(real_traits<float>::rsq(r2.x), real_traits<float>::rsq(r2.y)),
                         make_float2(s.w, s.w), acc);
      }
      acc = __fadd2_rn(acc, acc2);
      float fa = acc.x, fb = acc.y;
      for (int off = R; off < 32; off <<= 1) {
        fa += __shfl_xor_sync(kFull, fa, off);
        fb += __shfl_xor_sync(kFull, fb, off);
      }
      const float c = real_traits<float>::inv4pi();
      if (sub == 0) {
        if (live0) out[oa * nrhs + r] = fa * c + na * c;
        if (live1) out[ob * nrhs + r] = fb * c + nb * c;
      }
    }
  }
}

}  // namespace

extern "C" {

// Mutual near field into the partial-sum slots P (layout above); sources ==
// targets, tree order.  src4: (nrhs, npts) records (x, y, z, q); near_dst[e]
// = base_B + slot * n_B for an upper entry e of leaf A's near list (B > A),
// unused otherwise; P: nrhs planes of pstride floats.
int kifmm_p2p_mutual_f32(const float* tx, const float* ty, const float* tz, const int32_t* lstart,
                         const int32_t* lcount, int64_t n_leaves, const float* src4, int64_t npts,
                         const int32_t* near_off, const int32_t* near_leaf,
                         const int32_t* near_dst, const int32_t* base, int64_t nrhs,
                         int64_t pstride, int guard, float* P, void* stream) {
  if (n_leaves < 0 || npts < 0 || nrhs < 1 || pstride < npts) return KIFMM_EARG;
  if (n_leaves == 0) return 0;
  const auto* s4 = reinterpret_cast<const float4*>(src4);
  if (guard)
    p2p_mutual_kernel<true><<<ceil_div(n_leaves, kMW), 32 * kMW, 0, (cudaStream_t)stream>>>(
        tx, ty, tz, lstart, lcount, n_leaves, s4, npts, near_off, near_leaf, near_dst, base, nrhs,
        pstride, P);
  else
    p2p_mutual_kernel<false><<<ceil_div(n_leaves, kMW), 32 * kMW, 0, (cudaStream_t)stream>>>(
        tx, ty, tz, lstart, lcount, n_leaves, s4, npts, near_off, near_leaf, near_dst, base, nrhs,
        pstride, P);
  return launch_status();
}

// out[perm[i]] = L2P(i) + sum of i's near-field slots (slot order).
int kifmm_l2p_mutual_f32(const float* tx, const float* ty, const float* tz, const int32_t* ts,
                         const int32_t* tc, int64_t ntl, const double* centers,
                         const double* ebase, int64_t ne, const float* local, int64_t nrhs,
                         const int64_t* perm, const int32_t* base, const int32_t* nlow,
                         int64_t pstride, const float* P, float* out, void* stream) {
  if (ntl < 0 || ne < 1 || ne > 1024 || nrhs < 1) return KIFMM_EARG;
  if (ntl == 0) return 0;
  const size_t smem = (size_t)kLW * ne * sizeof(float4);
  set_max_smem((const void*)l2p_mutual_kernel, smem);
  l2p_mutual_kernel<<<ceil_div(ntl, kLW), 32 * kLW, smem, (cudaStream_t)stream>>>(
      tx, ty, tz, ts, tc, ntl, centers, ebase, (int)ne, local, nrhs, perm, base, nlow, pstride, P,
      out);
  return launch_status();
}

}  // extern "C"
