// Factored float64 BLAS-M2L sweep on the FP64 tensor cores (DMMA).
//
// The reference applies, per transfer vector t, (q~[rows_s] . vbar_t) . ubar_t^T
// (m2l_blas.py:291-320): 4 k k_t flop per pair.  The dense sweep of
// m2l_blas.cu contracts D_t = ubar_t vbar_t^T once and spends 2 k^2 per pair -
// twice the work and more when k_t << k (config 4 float64: k = 147, mean
// k_t = 24; config 5: k = 483, mean k_t = 93).  Here the two factors are
// applied in two passes with the k_t-wide intermediate in HBM:
//
//   compress  W[pair] = q~[src(pair)] . vbar_t          (K = k,   N = k_t)
//             bucket-stationary: a CTA takes 128 pairs of ONE vector t - dense
//             row chunks even on sparse trees - and streams K in BK-chunks.
//   expand    acc[target] += W[pair(target, t)] . ubar_t^T   (K = k_t, N = k)
//             target-stationary like the dense sweep: a CTA owns a tile of 128
//             same-class targets, walks its vectors, and each vector
//             contributes K = k_t (padded to 16) instead of k.
//
// Both passes are the same pipelined DMMA kernel (cp.async ring of STG
// stages, mma.sync m8n8k4 f64, 8 warps = 4 row blocks x 2 column halves, a
// warp owns 32 x 8 NTW accumulator columns); they differ in where a step's
// rows, operator and K come from.  No atomics: every W row and every
// accumulator row has one writer; the vector-range split of the expand pass
// writes separate column blocks that the following GEMM sums in a fixed
// order, as for the dense sweep.
//
// Layouts: vbar (316 blocks, block t = (kin x ktp_t) row-major at voff[t]),
// ubar^T (block t = (ktp_t x ko_pad) row-major at uoff[t]), ktp_t = k_t padded
// (a multiple of 16; of 16 * slabs above 160), rows/columns beyond k / k_t
// zero.  W: per vector t a block of (pairs of t, padded to 128) x ktp_t at
// 16-byte offset wbase16[t]; one plane per right-hand side.
#include "common.cuh"

using namespace kifmm;

namespace {

constexpr int TMT = 128;

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

struct FactArgs {
  // rows of a step: compress -> q~ row (s*nrhs + r)*kin; expand -> W + off16*2
  const double* A;
  int64_t a_plane;                 // expand: elements between the rhs planes of W
  int kin;                         // compress: K and q~ row length
  const double* B;                 // vbar / ubar^T blocks
  const int64_t* boff;             // (316) element offset of block t
  const int32_t* ktp;              // (316) padded rank
  int ko_pad;                      // expand: row stride of ubar^T blocks and accumulator width
  // compress tiles
  const int32_t* tile_t;           // (n_tiles) vector of the tile
  const int32_t* tile_first;       // (n_tiles) first pair (within its vector) of the tile
  const int32_t* rows1;            // (n_tiles, 128) q~ row of each pair, -1 padding
  const int64_t* wbase16;          // (316) 16-byte offset of vector t's W block
  double* W;
  int64_t w_plane;
  // expand tiles
  const int32_t* tile_targets;     // (n_tiles, 128)
  const int32_t* tile_class;       // (n_tiles)
  const int32_t* woff;             // (n_tiles, 189, 128) 16-byte offset of the pair's W row, -1 none
  const int32_t* class_tv;         // (8, 189)
  const uint16_t* gmask;           // optional sparse lists (as m2l_blas.cu)
  const int16_t* jlist;
  const int32_t* jcount;
  int nsplit, jper, n_slabs;
  int64_t nrhs;
  double* acc;
};

template <int NTW, int BK, int STG, bool EXPAND>
__global__ void __launch_bounds__(256, 1) factored_dmma_kernel(const FactArgs a) {
  constexpr int GS = BK + 4;                          // conflict-free A fragment loads
  constexpr int KOB = 16 * NTW;
  // operator row stride = 4 mod 16 doubles: the 16 lanes of a half-warp read
  // rows (lane & 3), columns (lane >> 2) of a k4 x 8 fragment from 16 distinct
  // 8-byte bank pairs (KOB + 8 put rows k and k + 2 on the same banks)
  constexpr int DS = KOB + 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Gs = reinterpret_cast<double*>(smem_raw);   // [STG][TMT][GS]
  double* Ds = Gs + STG * TMT * GS;                   // [STG][BK][DS]
  __shared__ uint32_t stage_bits[STG];
  __shared__ int16_t vec_t[192];                      // vector of position p - j0
  __shared__ int16_t vec_j[192];                      // class-list index of position p - j0
  __shared__ uint8_t vec_ch[192];                     // K-chunks of position p - j0
  __shared__ int16_t vec_K[192];                      // K of position p - j0
  __shared__ int64_t vec_boff[192];                   // operator block offset of position p - j0
  __shared__ int nsteps_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;
  const int64_t tile = blockIdx.x;
  const int64_t r = blockIdx.y;
  const int slab = blockIdx.z % a.n_slabs, split = blockIdx.z / a.n_slabs;
  const int c0 = slab * KOB;

  // ---- the tile's steps: (vector, K) per position
  int j0 = 0, j1 = 1;
  const int32_t* tsrc = nullptr;
  const uint16_t* gm = nullptr;
  if (EXPAND) {
    const int cnt = a.jcount ? a.jcount[tile] : 189;
    const int jp = a.jcount ? (cnt + a.nsplit - 1) / a.nsplit : a.jper;
    j0 = split * jp;
    j1 = min(cnt, j0 + jp);
    tsrc = a.woff + tile * 189 * TMT;
    gm = a.gmask ? a.gmask + tile * 189 : nullptr;
  }
  if (tid == 0) nsteps_s = 0;
  __syncthreads();
  if (EXPAND) {
    const int32_t* tv_list = a.class_tv + a.tile_class[tile] * 189;
    const int16_t* jl = a.jlist ? a.jlist + tile * 189 : nullptr;
    int mine = 0;
    for (int p = j0 + tid; p < j1; p += 256) {
      const int j = jl ? (int)jl[p] : p;
      const int t = tv_list[j];
      const int K = a.ktp[t];
      const int ch = (K + BK - 1) / BK;
      vec_t[p - j0] = (int16_t)t;
      vec_j[p - j0] = (int16_t)j;
      vec_ch[p - j0] = (uint8_t)ch;
      vec_K[p - j0] = (int16_t)K;
      vec_boff[p - j0] = a.boff[t];
      mine += ch;
    }
    if (mine) atomicAdd(&nsteps_s, mine);
  } else if (tid == 0) {
    const int t = a.tile_t[tile];
    vec_t[0] = (int16_t)t;
    vec_j[0] = 0;
    vec_ch[0] = (uint8_t)((a.kin + BK - 1) / BK);
    vec_K[0] = (int16_t)a.ktp[t];                     // compress: the tile's width (ldb, ldw)
    vec_boff[0] = a.boff[t];
    nsteps_s = (a.kin + BK - 1) / BK;
  }
  __syncthreads();
  const int nsteps = nsteps_s;
  if (!EXPAND && c0 >= vec_K[0]) return;               // (never: tiles are grouped by width)

  double acc[4][NTW][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NTW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // gather assignment: 16-byte chunk tid % CPR of rows tid / CPR + RPP * i
  constexpr int CPR = BK / 2, RPP = 256 / CPR, NR = TMT / RPP;
  const int grow = tid / CPR, gch = tid % CPR;
  int ids_cur[NR], ids_next[NR];
  auto load_ids = [&](int pos, int (&ids)[NR]) {          // pos = position - j0
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      if (EXPAND)
        ids[i] = pos < j1 - j0 ? __ldg(&tsrc[(int)vec_j[pos] * TMT + grow + RPP * i]) : -1;
      else
        ids[i] = pos == 0 ? __ldg(&a.rows1[tile * TMT + grow + RPP * i]) : -1;
    }
  };
  int sp = 0, sch = 0;                                 // staging cursor: position - j0, chunk
  auto stage = [&](int buf) {
    if (sch == 0) {
#pragma unroll
      for (int i = 0; i < NR; ++i) ids_cur[i] = ids_next[i];
      load_ids(sp + 1, ids_next);
    }
    // (per-vector K and operator offset come from shared memory: no dependent
    // global loads in front of the cp.async issue)
    const int K = EXPAND ? (int)vec_K[sp] : a.kin;
    if (tid == 0) stage_bits[buf] = gm ? (uint32_t)gm[vec_j[sp]] : 0xFFFFu;
    const int kk0 = sch * BK;
    const bool k_ok = kk0 + 2 * gch < K;               // a partial last chunk reads zeros
    double* g = Gs + buf * TMT * GS;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int s = ids_cur[i];
      const bool ok = s >= 0 && k_ok;
      const double* gp;
      if (EXPAND)
        gp = a.A + r * a.a_plane + (ok ? (int64_t)s * 2 + kk0 + 2 * gch : 0);
      else
        gp = a.A + (ok ? ((int64_t)s * a.nrhs + r) * a.kin + kk0 + 2 * gch : 0);
      cp_async16(g + (grow + RPP * i) * GS + 2 * gch, gp, ok);
    }
    const int ldb = EXPAND ? a.ko_pad : (int)vec_K[0];
    const double* bsrc = a.B + vec_boff[sp] + (int64_t)kk0 * ldb + c0;
    double* d = Ds + buf * BK * DS;
    constexpr int DCH = BK * KOB / 2;
    for (int e = tid; e < DCH; e += 256) {
      const int row = e / (KOB / 2), v = e - row * (KOB / 2);
      const bool ok = kk0 + row < K;
      cp_async16(d + row * DS + 2 * v, ok ? bsrc + (int64_t)row * ldb + 2 * v : a.B, ok);
    }
    cp_async_commit();
    if (++sch == (int)vec_ch[sp]) {
      sch = 0;
      ++sp;
    }
  };

  load_ids(0, ids_next);
  for (int q = 0; q < STG - 1; ++q) {
    if (q < nsteps) stage(q);
    else cp_async_commit();
  }
  const int arow = 32 * wm + (lane >> 2), acol = lane & 3;
  const int bcol = wn * (KOB / 2) + (lane >> 2), brow = lane & 3;
  for (int st = 0; st < nsteps; ++st) {
    const int buf = st % STG;
    cp_async_wait<STG - 2>();
    __syncthreads();
    if (st + STG - 1 < nsteps) stage((st + STG - 1) % STG);
    else cp_async_commit();
    const double* g = Gs + buf * TMT * GS + arow * GS + acol;
    const double* d = Ds + buf * BK * DS + brow * DS + bcol;
    const uint32_t mb = (stage_bits[buf] >> (4 * wm)) & 0xFu;   // warp-uniform
    if (mb == 0xFu) {
#pragma unroll
      for (int ks = 0; ks < BK; ks += 4) {
        double av[4], bv[NTW];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) av[mt] = g[mt * 8 * GS + ks];
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt) bv[nt] = d[ks * DS + nt * 8];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) dmma884(acc[mt][nt], av[mt], bv[nt]);
      }
    } else if (mb) {
#pragma unroll 2
      for (int ks = 0; ks < BK; ks += 4) {
        double bv[NTW];
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt) bv[nt] = d[ks * DS + nt * 8];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          if (!((mb >> mt) & 1u)) continue;
          const double av = g[mt * 8 * GS + ks];
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) dmma884(acc[mt][nt], av, bv[nt]);
        }
      }
    }
  }
  cp_async_wait<0>();

  if (EXPAND) {
    const int64_t ld = (int64_t)a.nsplit * a.ko_pad;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int32_t tgt = a.tile_targets[tile * TMT + 32 * wm + 8 * mt + (lane >> 2)];
      if (tgt < 0) continue;
      double* o = a.acc + ((int64_t)tgt * a.nrhs + r) * ld + (int64_t)split * a.ko_pad + c0 +
                  wn * (KOB / 2) + 2 * (lane & 3);
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt)
        *reinterpret_cast<double2*>(o + nt * 8) = double2{acc[mt][nt][0], acc[mt][nt][1]};
    }
  } else {
    const int t = vec_t[0];
    const int64_t ldw = vec_K[0];
    double* base = a.W + r * a.w_plane + a.wbase16[t] * 2;
    const int64_t first = a.tile_first[tile];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int m = 32 * wm + 8 * mt + (lane >> 2);
      // padding rows of the last tile of a vector are inside its W block
      double* o = base + (first + m) * ldw + c0 + wn * (KOB / 2) + 2 * (lane & 3);
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt)
        *reinterpret_cast<double2*>(o + nt * 8) = double2{acc[mt][nt][0], acc[mt][nt][1]};
    }
  }
}

template <int NTW, int BK, int STG, bool EXPAND>
int launch_fact(const FactArgs& a, dim3 grid, cudaStream_t s) {
  const size_t smem = sizeof(double) * (size_t)STG * (TMT * (BK + 4) + BK * (16 * NTW + 4));
  auto k = factored_dmma_kernel<NTW, BK, STG, EXPAND>;
  set_max_smem((const void*)k, smem);
  k<<<grid, 256, smem, s>>>(a);
  return launch_status();
}

template <bool EXPAND>
int dispatch(int ntw, const FactArgs& a, dim3 grid, cudaStream_t s) {
  // expand: K = k_t (padded to 16) in 32-wide chunks and 3 stages up to 128
  // accumulator columns (config 5: 73 vs 80 ms), 16-wide chunks and 4 stages
  // above (three 32-wide stages do not fit; two measured slower, config 4:
  // 37 vs 33 ms).
  // compress: K = k in 32-wide chunks; 3 stages where they fit the 227 KB
  // (widths 80..128), 2 stages for the widest tiles, and 2 stages for narrow
  // tiles (<= 64 columns) so that two CTAs share an SM
#define KIFMM_FACT(NT_)                                                         \
  case NT_:                                                                     \
    if (EXPAND)                                                                 \
      return NT_ <= 8 ? launch_fact<NT_, 32, 3, true>(a, grid, s)               \
                      : launch_fact<NT_, 16, 4, true>(a, grid, s);              \
    if (NT_ >= 5 && NT_ <= 8) return launch_fact<NT_, 32, 3, false>(a, grid, s); \
    return launch_fact<NT_, 32, 2, false>(a, grid, s);
  switch (ntw) {
    KIFMM_FACT(1) KIFMM_FACT(2) KIFMM_FACT(3) KIFMM_FACT(4) KIFMM_FACT(5)
    KIFMM_FACT(6) KIFMM_FACT(7) KIFMM_FACT(8) KIFMM_FACT(9) KIFMM_FACT(10)
  }
#undef KIFMM_FACT
  return KIFMM_EARG;
}

}  // namespace

extern "C" {

// Compress pass of the factored float64 BLAS-M2L (m2l_blas.py:291-305, first
// factor): for the n_tiles 128-pair chunks of ONE width class (every tile's
// vector has ktp = 16 * ntw * n_slabs), W[pair] = q~[rows1[pair]] . vbar_t.
int kifmm_m2l_compress_f64(const double* qt, int64_t kin, int64_t nrhs, const double* vbar,
                           const int64_t* voff, const int32_t* ktp, const int32_t* tile_t,
                           const int32_t* tile_first, const int32_t* rows1, int64_t n_tiles,
                           int64_t ntw, int64_t n_slabs, const int64_t* wbase16, double* W,
                           int64_t w_plane, void* stream) {
  if (kin < 16 || kin % 2 || nrhs < 1 || n_tiles < 0 || ntw < 1 || ntw > 10 || n_slabs < 1)
    return KIFMM_EARG;
  if (n_tiles == 0) return 0;
  FactArgs a = {};
  a.A = qt;
  a.kin = (int)kin;
  a.nrhs = nrhs;
  a.B = vbar;
  a.boff = voff;
  a.ktp = ktp;
  a.tile_t = tile_t;
  a.tile_first = tile_first;
  a.rows1 = rows1;
  a.wbase16 = wbase16;
  a.W = W;
  a.w_plane = w_plane;
  a.n_slabs = (int)n_slabs;
  a.nsplit = 1;
  dim3 grid((unsigned)n_tiles, (unsigned)nrhs, (unsigned)n_slabs);
  return dispatch<false>((int)ntw, a, grid, (cudaStream_t)stream);
}

// Expand pass (second factor, m2l_blas.py:306-320 without the scatter):
// acc[target] += sum over the tile's vectors of W[pair] . ubar_t^T; the same
// tile plan, vector split and sparse lists as kifmm_m2l_sweep_sparse_f64.
int kifmm_m2l_expand_f64(const double* W, int64_t w_plane, const double* ubT, const int64_t* uoff,
                         const int32_t* ktp, int64_t ko_pad, const int32_t* tile_targets,
                         const int32_t* tile_class, const int32_t* woff, const int32_t* class_tv,
                         int64_t n_tiles, int64_t nrhs, int64_t nsplit, const uint16_t* gmask,
                         const int16_t* jlist, const int32_t* jcount, double* acc, void* stream) {
  constexpr int KOB_MAX = 160;
  if (ko_pad < 16 || n_tiles < 0 || nrhs < 1 || nsplit < 1 || nsplit > 189) return KIFMM_EARG;
  if ((gmask || jlist || jcount) && !(gmask && jlist && jcount)) return KIFMM_EARG;
  if (n_tiles == 0) return 0;
  const int n_slabs = (int)((ko_pad + KOB_MAX - 1) / KOB_MAX);
  if (ko_pad % n_slabs) return KIFMM_EARG;
  const int kob = (int)(ko_pad / n_slabs);
  if (kob % 16 || kob > KOB_MAX) return KIFMM_EARG;
  FactArgs a = {};
  a.A = W;
  a.a_plane = w_plane;
  a.nrhs = nrhs;
  a.B = ubT;
  a.boff = uoff;
  a.ktp = ktp;
  a.ko_pad = (int)ko_pad;
  a.tile_targets = tile_targets;
  a.tile_class = tile_class;
  a.woff = woff;
  a.class_tv = class_tv;
  a.gmask = gmask;
  a.jlist = jlist;
  a.jcount = jcount;
  a.nsplit = (int)nsplit;
  a.jper = (int)((189 + nsplit - 1) / nsplit);
  a.n_slabs = n_slabs;
  a.acc = acc;
  dim3 grid((unsigned)n_tiles, (unsigned)nrhs, (unsigned)(n_slabs * nsplit));
  return dispatch<true>(kob / 16, a, grid, (cudaStream_t)stream);
}

}  // extern "C"
