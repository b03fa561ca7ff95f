/*
 * kifmm_b200.h - C ABI of the B200 (sm_100a) kiFMM hot path.
 *
 * All entry points are extern "C", take DEVICE pointers plus sizes and a
 * CUDA stream handle (cudaStream_t passed as void*), never allocate, and
 * return an int status: 0 = ok, KIFMM_EARG (10001) = bad argument,
 * otherwise the cudaError_t of the launch.  Buffers are C-contiguous.
 * "accumulate" outputs follow the reference semantics (+=).
 *
 * Two groups:
 *  (1) the reference's native plug-in boundary, one function per loop of
 *      kifmm3d/_hot.pyx, bound in the reference through hotloops.py;
 *  (2) the level/leaf passes the reference runs through numpy inside
 *      engine.evaluate (engine.py:270-404), which the device engine chains
 *      without host round trips.
 */
#ifndef KIFMM_B200_H
#define KIFMM_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KIFMM_EARG 10001

/* ---- (1) kernel-level boundary ------------------------------------------ */

/* Replaces _hot.laplace_potentials (_hot.pyx:24-65, bound at hotloops.py:54-57):
 * out[i, r] += sum_j K(t_i, s_j) * charges[j, r], K = 1/(4 pi r), 0 if r == 0. */
int kifmm_laplace_potentials_f32(const float* tx, const float* ty, const float* tz, int64_t nt,
                                 const float* sx, const float* sy, const float* sz, int64_t ns,
                                 const float* charges, int64_t nrhs, float* out, void* stream);
int kifmm_laplace_potentials_f64(const double* tx, const double* ty, const double* tz, int64_t nt,
                                 const double* sx, const double* sy, const double* sz, int64_t ns,
                                 const double* charges, int64_t nrhs, double* out, void* stream);

/* Extension (no reference counterpart: the reference is potential-only;
 * BASELINE config 3 asks for potential and gradient): direct sum of both,
 * phi[i, r] += sum_j K q_j, grad[i, r, :] += sum_j q_j grad_t K(t_i, s_j)
 * = -sum_j q_j (t_i - s_j) / (4 pi r^3), pairs with r == 0 skipped. */
int kifmm_laplace_gradients_f32(const float* tx, const float* ty, const float* tz, int64_t nt,
                                const float* sx, const float* sy, const float* sz, int64_t ns,
                                const float* charges, int64_t nrhs, float* phi, float* grad,
                                void* stream);
int kifmm_laplace_gradients_f64(const double* tx, const double* ty, const double* tz, int64_t nt,
                                const double* sx, const double* sy, const double* sz, int64_t ns,
                                const double* charges, int64_t nrhs, double* phi, double* grad,
                                void* stream);

/* Replaces _hot.laplace_matrix (_hot.pyx:68-88, hotloops.py:60-64): out[i, j] = K(t_i, s_j). */
int kifmm_laplace_matrix_f32(const float* tx, const float* ty, const float* tz, int64_t nt,
                             const float* sx, const float* sy, const float* sz, int64_t ns,
                             float* out, void* stream);
int kifmm_laplace_matrix_f64(const double* tx, const double* ty, const double* tz, int64_t nt,
                             const double* sx, const double* sy, const double* sz, int64_t ns,
                             double* out, void* stream);

/* Replaces _hot.p2p_blocked (_hot.pyx:91-138, hotloops.py:67-71): target i sums
 * the gathered sources src_offsets[b] .. src_offsets[b+1] of its leaf
 * b = leaf_of_target[i]; out[i, r] += that sum. */
int kifmm_p2p_blocked_f32(const float* tx, const float* ty, const float* tz, int64_t nt,
                          const int64_t* leaf_of_target, const float* sx, const float* sy,
                          const float* sz, const float* charges, int64_t nrhs,
                          const int64_t* src_offsets, int64_t n_leaves, float* out, void* stream);
int kifmm_p2p_blocked_f64(const double* tx, const double* ty, const double* tz, int64_t nt,
                          const int64_t* leaf_of_target, const double* sx, const double* sy,
                          const double* sz, const double* charges, int64_t nrhs,
                          const int64_t* src_offsets, int64_t n_leaves, double* out, void* stream);

/* Replaces _hot.hadamard_m2l (_hot.pyx:141-178, hotloops.py:74-77), complex
 * interleaved (re, im):
 * phat[f, c, tau, r] += sum_o sum_sigma khat[f, o, tau, sigma] * qhat[f, halo[c, o], sigma, r]
 * khat (nf, 26, 8, 8), qhat (nf, nsc, 8, nrhs), halo (ntc, 26) (-1 = absent),
 * phat (nf, ntc, 8, nrhs). */
int kifmm_hadamard_m2l_c64(const float* khat, const float* qhat, const int64_t* halo, float* phat,
                           int64_t nf, int64_t nsc, int64_t ntc, int64_t nrhs, void* stream);
int kifmm_hadamard_m2l_c128(const double* khat, const double* qhat, const int64_t* halo,
                            double* phat, int64_t nf, int64_t nsc, int64_t ntc, int64_t nrhs,
                            void* stream);

/* The same product over a tile plan of the halo table (m2l_fft.py
 * plan_hadamard_tiles): tile t owns target clusters [tile_begin[t],
 * tile_begin[t+1]); tcol (n_tiles, 256) int16 = tile-local target of each
 * slot-table column (-1 = empty; column 32w + 4g + j holds a target of
 * coordinate parity class g); src[src_off[t] .. src_off[t+1]) = source
 * cluster of each shared-memory slot (at most 600, -1 = hole, slot % 8 =
 * the source's parity class); slots (n_tiles, 26, 256) int16 = slot of
 * (offset, column), 600 + class = absent.  Each frequency's sources are
 * staged once per tile.  accumulate = 0 stores (phat need not be zeroed),
 * 1 adds. */
int kifmm_hadamard_tiled_c64(const float* khat, const float* qhat, const int64_t* tile_begin,
                             const int64_t* src_off, const int64_t* src, const int16_t* slots,
                             const int16_t* tcol, int64_t n_tiles, int64_t nf, int64_t nsc,
                             int64_t ntc, int64_t nrhs, int accumulate, float* phat, void* stream);
int kifmm_hadamard_tiled_c128(const double* khat, const double* qhat, const int64_t* tile_begin,
                              const int64_t* src_off, const int64_t* src, const int16_t* slots,
                              const int16_t* tcol, int64_t n_tiles, int64_t nf, int64_t nsc,
                              int64_t ntc, int64_t nrhs, int accumulate, double* phat,
                              void* stream);

/* ---- (2) engine passes (device-resident evaluate) ------------------------ */

/* Row-major C[rowmap(m), n] (=|+=) alpha * sum_k A'[m, k] B[k, n] * colscale[n],
 * A'[m, k] = sum_{s < asum} A[m*lda + s*astride + k] (asum = 1: plain A).
 * rowmap NULL -> identity; rowmap[m] < 0 -> row skipped.  colscale may be NULL.
 * Used for the projection/expansion of BLAS-M2L (m2l_blas.py:285,322; the
 * A-sum reduces the split sweep's partial accumulators), the factored
 * pseudo-inverse solves (expansion.py:78-82) and the M2M/L2L products. */
int kifmm_gemm_f32(int64_t M, int64_t N, int64_t K, float alpha, const float* A, int64_t lda,
                   int asum, int64_t astride, const float* B, int64_t ldb, const float* colscale,
                   float* C, int64_t ldc, const int32_t* rowmap, int accumulate, void* stream);
int kifmm_gemm_f64(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                   int asum, int64_t astride, const double* B, int64_t ldb,
                   const double* colscale, double* C, int64_t ldc, const int32_t* rowmap,
                   int accumulate, void* stream);

/* Fused operator chain on row tiles (csrc/chain.cu):
 *   Y0 = X . B0 * cs0 * al0;  Y(s) = Y(s-1) re-read as rows of width K(s) . B(s) * cs(s) * al(s)
 *   C[rowmap(row)] (=|+=) Y(last)
 * X rows: A[m*lda + k] summed over asum blocks (stride astride), or, when
 * a_child is set, the 8 child rows a_child[p*8+c]*a_nrhs + r concatenated
 * (M2M stacking).  B(s) are (K(s) x N(s)) row-major; cs(s) may be NULL.
 * Used for the P2M solve, M2M, the M2L expansion + check->local solve and
 * L2L (kernel product, then the factored pseudo-inverse, as the reference). */
int kifmm_chain_f32(int64_t M, const float* A, int64_t lda, int asum, int64_t astride,
                    const int32_t* a_child, int64_t child_w, int64_t a_nrhs, int nstage,
                    const float* B0, const float* B1, const float* B2, int64_t K0, int64_t N0,
                    int64_t K1, int64_t N1, int64_t K2, int64_t N2, const float* cs0,
                    const float* cs1, const float* cs2, double al0, double al1, double al2,
                    float* C, int64_t ldc, const int32_t* c_rowmap, int accumulate, void* stream);
int kifmm_chain_f64(int64_t M, const double* A, int64_t lda, int asum, int64_t astride,
                    const int32_t* a_child, int64_t child_w, int64_t a_nrhs, int nstage,
                    const double* B0, const double* B1, const double* B2, int64_t K0, int64_t N0,
                    int64_t K1, int64_t N1, int64_t K2, int64_t N2, const double* cs0,
                    const double* cs1, const double* cs2, double al0, double al1, double al2,
                    double* C, int64_t ldc, const int32_t* c_rowmap, int accumulate,
                    void* stream);

/* P2M check potentials (engine.py:298-319): for source leaf l and check point c,
 * phi[(l*nrhs + r)*nc + c] = sum_{j in leaf} K(center_l + base_c, s_j) q[j*nrhs + r];
 * centers (n_leaves, 3) and base (nc, 3) are float64, summed exactly then rounded. */
int kifmm_p2m_check_f32(const float* sx, const float* sy, const float* sz, const float* q,
                        int64_t nrhs, const int32_t* leaf_start, const int32_t* leaf_count,
                        int64_t n_leaves, const double* centers, const double* base, int64_t nc,
                        float* phi, void* stream);
int kifmm_p2m_check_f64(const double* sx, const double* sy, const double* sz, const double* q,
                        int64_t nrhs, const int32_t* leaf_start, const int32_t* leaf_count,
                        int64_t n_leaves, const double* centers, const double* base, int64_t nc,
                        double* phi, void* stream);

/* M2M child stacking (engine.py:321-334): out[(p*nrhs + r), c*ne + e] =
 * mult[(child[p*8+c]*nrhs + r)*ne + e] or 0 where child < 0. */
int kifmm_stack_children_f32(const float* mult, const int32_t* child, int64_t n_par, int64_t nrhs,
                             int64_t ne, float* out, void* stream);
int kifmm_stack_children_f64(const double* mult, const int32_t* child, int64_t n_par,
                             int64_t nrhs, int64_t ne, double* out, void* stream);

/* BLAS-M2L fused bucket sweep (m2l_blas.py:284-320), target-stationary:
 * acc[(tgt*nrhs + r), p*ko + a] = sum_{j in piece p} sum_b Dt[tv(j), b, a] qt[(src*nrhs + r)*ki + b]
 * over the 189 vectors j of each tile's parity class (ascending), split into
 * nsplit contiguous pieces p (row stride nsplit*ko); the caller sums the
 * pieces (the expansion GEMM does, in fixed order).
 * qt (n_src*nrhs, ki) zero-padded; Dt (316, ki, ko) transposed dense cores.
 * tile_targets (n_tiles*128), tile_class (n_tiles), src (n_tiles, 189, 128),
 * class_tv (8, 189).  Padding slots (target -1) are skipped. */
int kifmm_m2l_sweep_f32(const float* qt, const float* Dt, int64_t ki, int64_t ko,
                        const int32_t* tile_targets, const int32_t* tile_class,
                        const int32_t* src, const int32_t* class_tv, int64_t n_tiles,
                        int64_t nrhs, int64_t nsplit, float* acc, void* stream);
int kifmm_m2l_sweep_f64(const double* qt, const double* Dt, int64_t ki, int64_t ko,
                        const int32_t* tile_targets, const int32_t* tile_class,
                        const int32_t* src, const int32_t* class_tv, int64_t n_tiles,
                        int64_t nrhs, int64_t nsplit, double* acc, void* stream);
/* float64 sweep for sparse trees (empty boxes skipped, config 5): per tile
 * only the vectors jlist[tile][0 .. jcount[tile]) that meet a source (int16,
 * ascending), and per vector the 8-row groups with a source (gmask bits,
 * uint16 over the tile's 16 groups); the others skip their DMMAs. */
int kifmm_m2l_sweep_sparse_f64(const double* qt, const double* Dt, int64_t kin, int64_t ko_pad,
                               const int32_t* tile_targets, const int32_t* tile_class,
                               const int32_t* src, const int32_t* class_tv, int64_t n_tiles,
                               int64_t nrhs, int64_t nsplit, const uint16_t* gmask,
                               const int16_t* jlist, const int32_t* jcount, double* acc,
                               void* stream);

/* Same sweep on the tcgen05 tensor cores for float32 (3xTF32): the caller
 * passes q~ split into TF32 hi/lo parts (kifmm_split_tf32) and the cores
 * split into hi/lo and packed per (vector, 32-wide K chunk) in the
 * canonical K-major UMMA layout [a/8][b/4][a%8][b%4] (device.py
 * pack_tc_cores).  kin % 8 == 0, n_out % 16 == 0, n_out <= 256.
 * acc layout as kifmm_m2l_sweep_f32 with ko = n_out. */
int kifmm_m2l_sweep_tc_f32(const float* qhi, const float* qlo, const float* bhi, const float* blo,
                           int64_t kin, int64_t n_out, const int32_t* tile_targets,
                           const int32_t* tile_class, const int32_t* src, const int32_t* class_tv,
                           int64_t n_tiles, int64_t nrhs, int64_t nsplit, float* acc, void* stream);

/* TMA-fed variant for the engine (csrc/m2l_tma.cu): q~ hi/lo live in dense
 * parity sub-lattice arrays (8*nrhs, h, h, h, kin) (kifmm_dense_split_tf32);
 * tile_ids (n_tiles) select class tiles of 4x4x8 same-parity targets
 * (class-major, then x, y, z tile index), tile_targets (n_tiles*128) map each
 * tile row (x*32 + y*8 + z) to a target row or -1; offsets (316, 3) int8 are
 * the transfer vectors.  kin % 8 == 0 and kin <= 128. */
int kifmm_m2l_sweep_tma_f32(const float* qhi, const float* qlo, const float* bhi, const float* blo,
                            int64_t kin, int64_t n_out, int64_t h, const int32_t* tile_targets,
                            const int32_t* tile_ids, int64_t n_tiles, const int32_t* class_tv,
                            const int8_t* offsets, int64_t nrhs, int64_t nsplit, float* acc,
                            void* stream);

/* Tensor-memory variant (csrc/m2l_tmem.cu), persistent, one CTA per SM:
 * the same tiles and dense sub-lattice array, but q (8*nrhs, h, h, h, kp)
 * holds RAW fp32 q~ (kifmm_dense_split_tf32 with lo == NULL); each target
 * row's source row is loaded into registers, split into TF32 hi/lo and
 * stored into TMEM as the MMA's A operand.  bpair (316, 2*kp*kp) is
 * [B_hi | B_lo] per vector, each packed [a/8][b/4][a%8][b%4] with one
 * K chunk of width kp (device.py pack_tmem_cores).  class_tv (8, 189) may
 * list each class's vectors in any order (device.py uses a locality order).
 * Persistent, one CTA per SM over (rhs, tile, vector split) items; two
 * loader/MMA groups per CTA take alternate vectors (pairs / n_pairs are
 * accepted for ABI stability).
 * Output: acc[(tgt*nrhs + r)*(nsplit*ostride) + split*ostride + c], c < kp:
 * the caller sums the nsplit slots.
 * kp % 8 == 0, 8 <= kp <= 64, ostride >= kp, ostride % 4 == 0.  Replaces,
 * with m2l_sweep_tma, the bucket loop of m2l_blas.py:296-318. */
int kifmm_m2l_sweep_tmem_f32(const float* q, const float* bpair, int64_t kp, int64_t h,
                             const int32_t* tile_targets, const int32_t* tile_ids, int64_t n_tiles,
                             const int32_t* pairs, int64_t n_pairs, const int32_t* class_tv,
                             const int8_t* offsets, int64_t nrhs, int64_t nsplit, int64_t ostride,
                             float* acc, void* stream);

/* nsplit for kifmm_m2l_sweep_tmem_f32 that balances the persistent CTA pairs. */
int kifmm_m2l_sweep_tmem_splits(int64_t n_tiles, int64_t n_pairs, int64_t nrhs, int64_t* nsplit);

/* Debug timeline: clock64 stamps of CTA 0 of the following tensor-memory
 * sweeps with sub-lattice size h written into buf (12 x 1024 int64, device
 * memory); NULL disables. */
int kifmm_m2l_sweep_tmem_trace(long long* buf, int64_t h);

/* q~ rows (n_boxes*nrhs, kin) -> TF32 hi/lo parts scattered into the dense
 * sub-lattice arrays at slot[box] = parity*h^3 + (ix*h + iy)*h + iz. */
int kifmm_dense_split_tf32(const float* qt, const int32_t* slot, int64_t n_boxes, int64_t nrhs,
                           int64_t kin, int64_t h, float* hi, float* lo, void* stream);

/* x = hi + lo with hi, lo TF32 (cvt.rna.tf32.f32), elementwise. */
int kifmm_split_tf32(const float* x, int64_t n, float* hi, float* lo, void* stream);

/* FFT-M2L forward (m2l_fft.py:236-247): embed each box's multipole at
 * lattice+p of the n^3 grid (n = 2p), real 3-D DFT, and write the spectrum
 * frequency-major into qhat[(f*nsc + cluster)*8 + child)*nrhs + r] (complex).
 * slot_box (nsc*8): box row of each cluster slot or -1 (zero spectrum).
 * cluster_list (n_list) restricts the transform to those clusters (NULL = all). */
int kifmm_fft_forward_f32(const float* mult, int64_t nrhs, int64_t order, const int32_t* slot_box,
                          int64_t nsc, const int32_t* cluster_list, int64_t n_list, float* qhat,
                          void* stream);
int kifmm_fft_forward_f64(const double* mult, int64_t nrhs, int64_t order,
                          const int32_t* slot_box, int64_t nsc, const int32_t* cluster_list,
                          int64_t n_list, double* qhat, void* stream);

/* Factored float64 BLAS-M2L sweep (reference m2l_blas.py:291-320 applies
 * (q~[rows_s] vbar_t) ubar_t^T per bucket: 4 k k_t flop per pair; the dense
 * sweep above spends 2 k^2).  Two passes over an HBM intermediate W:
 * compress: W[pair] = q~[rows1[pair]] . vbar_t for the n_tiles 128-pair chunks
 *   of one width class (ktp_t = 16 * ntw * n_slabs); vbar block t = (kin x ktp_t)
 *   at voff[t]; W block t at 16-byte offset wbase16[t], one plane (w_plane
 *   elements) per right-hand side.
 * expand: acc[target] += sum_t W[pair(target, t)] . ubar_t^T, target-stationary
 *   on the tile plan of kifmm_m2l_sweep_f64 (woff: 16-byte W offset per
 *   (tile, vector position, row), -1 none; ubar^T block t = (ktp_t x ko_pad) at
 *   uoff[t]); optional sparse lists as kifmm_m2l_sweep_sparse_f64. */
int kifmm_m2l_compress_f64(const double* qt, int64_t kin, int64_t nrhs, const double* vbar,
                           const int64_t* voff, const int32_t* ktp, const int32_t* tile_t,
                           const int32_t* tile_first, const int32_t* rows1, int64_t n_tiles,
                           int64_t ntw, int64_t n_slabs, const int64_t* wbase16, double* W,
                           int64_t w_plane, void* stream);
int kifmm_m2l_expand_f64(const double* W, int64_t w_plane, const double* ubT, const int64_t* uoff,
                         const int32_t* ktp, int64_t ko_pad, const int32_t* tile_targets,
                         const int32_t* tile_class, const int32_t* woff, const int32_t* class_tv,
                         int64_t n_tiles, int64_t nrhs, int64_t nsplit, const uint16_t* gmask,
                         const int16_t* jlist, const int32_t* jcount, double* acc, void* stream);

/* Fused row chain for tall inputs (float32, operator dimensions <= 64):
 * Y0 = X B0 (x cs0, x al0), Y1 = Y0 B1 ..., with an optional output after every
 * stage (C_s, ldc_s, optional int32 row map over the M input rows - negative:
 * skipped -, accumulate flag); X[m][k] = sum_{s < asum} A[m*lda + s*astride + k].
 * The evaluate runs the P2M solve (expansion.py:78-82 via engine.py:298-318)
 * and the leaf level's M2L projection q~ = M S (m2l_blas.py:284-288) as one
 * launch: phi . U_up (x inv) . V_up^T (x side) -> multipoles, . S -> q~. */
int kifmm_rowchain_f32(int64_t M, const float* A, int64_t lda, int64_t asum, int64_t astride,
                       int64_t nstage, const float* B0, const float* B1, const float* B2,
                       int64_t K0, int64_t N0, int64_t N1, int64_t N2, const float* cs0,
                       const float* cs1, const float* cs2, float al0, float al1, float al2,
                       float* C0, float* C1, float* C2, int64_t ldc0, int64_t ldc1, int64_t ldc2,
                       const int32_t* map0, const int32_t* map1, const int32_t* map2, int64_t acc0,
                       int64_t acc1, int64_t acc2, void* stream);

/* Multipole halo pack/unpack for the multi-GPU exchange:
 * gather: dst[i*width + e] = src[rows[i]*width + e]; scatter: the reverse. */
int kifmm_gather_rows_f32(const float* src, const int32_t* rows, int64_t n_rows, int64_t width,
                          float* dst, void* stream);
int kifmm_gather_rows_f64(const double* src, const int32_t* rows, int64_t n_rows, int64_t width,
                          double* dst, void* stream);
int kifmm_scatter_rows_f32(const float* src, const int32_t* rows, int64_t n_rows, int64_t width,
                           float* dst, void* stream);
int kifmm_scatter_rows_f64(const double* src, const int32_t* rows, int64_t n_rows, int64_t width,
                           double* dst, void* stream);
/* dst[dst_rows[i]*width + e] = src[src_rows[i]*width + e]: the halo unpack of
 * the all-gathered exchange buffer (distributed.py; the reference has no
 * multi-GPU path, SPEC.md:139 - SURVEY 8(e)). */
int kifmm_move_rows_f32(const float* src, const int32_t* src_rows, const int32_t* dst_rows,
                        int64_t n_rows, int64_t width, float* dst, void* stream);
int kifmm_move_rows_f64(const double* src, const int32_t* src_rows, const int32_t* dst_rows,
                        int64_t n_rows, int64_t width, double* dst, void* stream);
/* dst[rows[i]*width + e] += src[i*width + e] (rows[i] < 0: skipped): the L2L
 * child check potentials added to the M2L check potentials of a level before
 * the one down_inv solve (engine.py:355,370 merged). */
int kifmm_scatter_add_rows_f32(const float* src, const int32_t* rows, int64_t n_rows,
                               int64_t width, float* dst, void* stream);
int kifmm_scatter_add_rows_f64(const double* src, const int32_t* rows, int64_t n_rows,
                               int64_t width, double* dst, void* stream);

/* FFT-M2L inverse (m2l_fft.py:252-261): for each target box b, take the
 * spectrum phat[f, tgt_slot[b], r], inverse real 3-D DFT, read the
 * lattice points and scale: check[(b*nrhs + r)*ne + e]. */
int kifmm_fft_inverse_f32(const float* phat, int64_t nrhs, int64_t order, const int32_t* slot_box,
                          int64_t ntc, double level_scale, float* check, void* stream);
int kifmm_fft_inverse_f64(const double* phat, int64_t nrhs, int64_t order,
                          const int32_t* slot_box, int64_t ntc, double level_scale, double* check,
                          void* stream);

/* Mutual near field, sources == targets (same tree), float32, potential.
 * Replaces _hot.p2p_blocked (_hot.pyx:91-138) on the gather plan of
 * engine.py:224-256 when the two clouds are one point set: each unordered
 * pair of adjacent leaves (A < B, Morton order) is evaluated once, one
 * rsqrt feeding both directions; the leaf's own block is direct (r2 == 0
 * -> 0).  Results go to partial-sum slots (no atomics, deterministic):
 *   P[r*pstride + base[B] + s*n_B + t], s = 0: B's row sums, s = 1..nlow_B:
 *   the column sums of B's s-th lower neighbour (its entry s of B's near list);
 * near_pack[e] = (start, count, dst, leaf) of entry e of a near list (the
 * CSR near_off): the entry leaf's first point and point count, and dst =
 * base[B] + s*n_B for an upper entry (A, B > A), base[A] for the own entry
 * (entry 0).  order (n_leaves, or NULL): the leaves in launch order
 * (heaviest first balances the uneven per-leaf work).  guard != 0: also
 * guard the cross-leaf pairs against r2 == 0. */
int kifmm_p2p_mutual_f32(const float* tx, const float* ty, const float* tz, int64_t n_leaves,
                         const float* src4, int64_t npts, const int32_t* near_off,
                         const int32_t* near_pack, const int32_t* order, int64_t nrhs,
                         int64_t pstride, int guard, float* P, void* stream);
int kifmm_p2p_mutual_f64(const double* tx, const double* ty, const double* tz, int64_t n_leaves,
                         const double* src4, int64_t npts, const int32_t* near_off,
                         const int32_t* near_pack, const int32_t* order, int64_t nrhs,
                         int64_t pstride, int guard, double* P, void* stream);
/* Near-field totals of the mutual pass: out[perm[i]*nrhs + r] = (1/4 pi)
 * sum_{s=0..nlow_b} P[r*pstride + base[b] + s*n_b + t] (slot order), for
 * target i = leaf b's t-th point; the L2P pass then accumulates onto out
 * (kifmm_leaf_pass_f32 with parts = 1 | 4). */
int kifmm_p2p_mutual_reduce_f32(const int32_t* tleaf_start, const int32_t* tleaf_count,
                                int64_t n_tleaves, int64_t nrhs, const int64_t* perm,
                                const int32_t* base, const int32_t* nlow, int64_t pstride,
                                const float* P, float* out, void* stream);
int kifmm_p2p_mutual_reduce_f64(const int32_t* tleaf_start, const int32_t* tleaf_count,
                                int64_t n_tleaves, int64_t nrhs, const int64_t* perm,
                                const int32_t* base, const int32_t* nlow, int64_t pstride,
                                const double* P, double* out, void* stream);
/* Potential + gradient variants (BASELINE config 3 asks for both; the reference
 * is potential-only): P holds four component planes per right-hand side
 * (potential, d/dx, d/dy, d/dz: P[(r*4 + c)*pstride + slot]); grad is
 * (target, rhs, 3) in the caller's order, like kifmm_leaf_pass_grad_*. */
int kifmm_p2p_mutual_grad_f32(const float* tx, const float* ty, const float* tz, int64_t n_leaves,
                              const float* src4, int64_t npts, const int32_t* near_off,
                              const int32_t* near_pack, const int32_t* order, int64_t nrhs,
                              int64_t pstride, int guard, float* P, void* stream);
int kifmm_p2p_mutual_grad_f64(const double* tx, const double* ty, const double* tz,
                              int64_t n_leaves, const double* src4, int64_t npts,
                              const int32_t* near_off, const int32_t* near_pack,
                              const int32_t* order, int64_t nrhs, int64_t pstride, int guard,
                              double* P, void* stream);
int kifmm_p2p_mutual_reduce_grad_f32(const int32_t* tleaf_start, const int32_t* tleaf_count,
                                     int64_t n_tleaves, int64_t nrhs, const int64_t* perm,
                                     const int32_t* base, const int32_t* nlow, int64_t pstride,
                                     const float* P, float* out, float* grad, void* stream);
int kifmm_p2p_mutual_reduce_grad_f64(const int32_t* tleaf_start, const int32_t* tleaf_count,
                                     int64_t n_tleaves, int64_t nrhs, const int64_t* perm,
                                     const int32_t* base, const int32_t* nlow, int64_t pstride,
                                     const double* P, double* out, double* grad, void* stream);

/* Leaf pass: fused L2P + P2P + un-permute (engine.py:377-404).  For target
 * leaf b and target i in it:
 *   out[perm[i]*nrhs + r] = sum_e K(t_i, center_b + base_e) local[(b*nrhs+r)*ne + e]
 *                         + sum_{near source leaves s of b, in order} sum_{j in s} K(t_i, s_j) q[j]
 * near_off (n_leaves+1) / near_leaf: source-leaf CSR (own leaf first, then
 * neighbours by Morton code, engine.py:231-240).  parts: bit 0 = L2P term,
 * bit 1 = P2P term, bit 2 = accumulate into out instead of overwriting,
 * bit 3 = guard every near-field record against r2 == 0 (not only the own
 * leaf's: set when float32 rounding merges points of different leaves);
 * perm NULL -> tree order. */
int kifmm_leaf_pass_f32(const float* tx, const float* ty, const float* tz, const int32_t* tleaf_start,
                        const int32_t* tleaf_count, int64_t n_tleaves, const double* centers,
                        const double* base, int64_t ne, const float* local, const float* src4,
                        int64_t ns, const int32_t* sleaf_start, const int32_t* sleaf_count,
                        const int32_t* near_off, const int32_t* near_leaf, int64_t nrhs,
                        const int64_t* perm, int parts, float* out, void* stream);
int kifmm_leaf_pass_f64(const double* tx, const double* ty, const double* tz,
                        const int32_t* tleaf_start, const int32_t* tleaf_count, int64_t n_tleaves,
                        const double* centers, const double* base, int64_t ne, const double* local,
                        const double* src4, int64_t ns, const int32_t* sleaf_start,
                        const int32_t* sleaf_count, const int32_t* near_off,
                        const int32_t* near_leaf, int64_t nrhs, const int64_t* perm, int parts,
                        double* out, void* stream);
/* Same pass with the potential gradient as well (config 3): grad[(perm[i] *
 * nrhs + r) * 3 + c] (=|+= with parts & 4) from the same L2P densities and
 * P2P sources.  grad must be non-NULL. */
int kifmm_leaf_pass_grad_f32(const float* tx, const float* ty, const float* tz,
                             const int32_t* tleaf_start, const int32_t* tleaf_count,
                             int64_t n_tleaves, const double* centers, const double* base,
                             int64_t ne, const float* local, const float* src4, int64_t ns,
                             const int32_t* sleaf_start, const int32_t* sleaf_count,
                             const int32_t* near_off, const int32_t* near_leaf, int64_t nrhs,
                             const int64_t* perm, int parts, float* out, float* grad,
                             void* stream);
int kifmm_leaf_pass_grad_f64(const double* tx, const double* ty, const double* tz,
                             const int32_t* tleaf_start, const int32_t* tleaf_count,
                             int64_t n_tleaves, const double* centers, const double* base,
                             int64_t ne, const double* local, const double* src4, int64_t ns,
                             const int32_t* sleaf_start, const int32_t* sleaf_count,
                             const int32_t* near_off, const int32_t* near_leaf, int64_t nrhs,
                             const int64_t* perm, int parts, double* out, double* grad,
                             void* stream);

/* Charge intake in one pass (engine.py:283-287: charges to tree order and the
 * working type) fused with the source pack below: qt[i*nrhs + r] =
 * (T) q_in[perm[i]*nrhs + r], src4[(r*n + i)*4 ..] = (x_i, y_i, z_i, q). */
int kifmm_gather_pack_f32(const double* q_in, const int64_t* perm, const float* sx,
                          const float* sy, const float* sz, int64_t n, int64_t nrhs, float* qt,
                          float* src4, void* stream);
int kifmm_gather_pack_f64(const double* q_in, const int64_t* perm, const double* sx,
                          const double* sy, const double* sz, int64_t n, int64_t nrhs, double* qt,
                          double* src4, void* stream);

/* L2P with an addend in tree order: out[perm[i]*nrhs + r] = addend[i*nrhs + r] +
 * sum_e K(t_i, center_b + base_e) local[(b*nrhs + r)*ne + e] (engine.py:377-389,
 * 399-404).  The overlapped evaluate passes the near-field totals
 * (kifmm_p2p_mutual_reduce_f32 with perm = NULL): both passes then touch the
 * totals coalesced and only the final store is permuted. */
int kifmm_l2p_add_f32(const float* tx, const float* ty, const float* tz, const int32_t* tleaf_start,
                      const int32_t* tleaf_count, int64_t n_tleaves, const double* centers,
                      const double* base, int64_t ne, const float* local, int64_t nrhs,
                      const int64_t* perm, const float* addend, float* out, void* stream);

/* AoS source records for the leaf pass (16/32-byte aligned):
 * src4[(r*ns + j)*4 + {0,1,2,3}] = (x_j, y_j, z_j, q[j*nrhs + r]). */
int kifmm_pack_sources_f32(const float* sx, const float* sy, const float* sz, const float* q,
                           int64_t ns, int64_t nrhs, float* src4, void* stream);
int kifmm_pack_sources_f64(const double* sx, const double* sy, const double* sz, const double* q,
                           int64_t ns, int64_t nrhs, double* src4, void* stream);

/* Charge intake: q_tree[i*nrhs + r] = (T) q_in[perm[i]*nrhs + r] (float64 in). */
int kifmm_gather_charges_f32(const double* q_in, const int64_t* perm, int64_t n, int64_t nrhs,
                             float* q_tree, void* stream);
int kifmm_gather_charges_f64(const double* q_in, const int64_t* perm, int64_t n, int64_t nrhs,
                             double* q_tree, void* stream);

/* Pipe-peak probe for roofline denominators: kind 0 FP32 FFMA, 1 FP64 DFMA,
 * 2 MUFU rsqrt; blocks*threads*iters*128 operations per launch. */
int kifmm_probe(int kind, int64_t blocks, int64_t threads, int64_t iters, void* out,
                void* stream);

/* Library identification: returns the compiled SM target (e.g. 100). */
int kifmm_sm_target(void);

/* ---- (5) device tree and plan build (octree.py:274-329,
 * engine.py:224-256, m2l_blas.py:232-258), bit-exact with the host build.
 * Codes are the reference's Morton keys: interleave(x, y, z) << 5 | level. */
/* Scratch bytes for op 0 = sort (incl. its index buffer), 1 = run-length
 * encode, 2 = unique; written to *bytes (host pointer). */
int kifmm_tree_temp_bytes(int op, int64_t n, int end_bit, int64_t* bytes);
/* Leaf codes of n points (n x 3 float64) in the domain (origin, side);
 * *bad (device int, zeroed by the caller) counts points outside it. */
int kifmm_tree_encode(const double* pts, int64_t n, double ox, double oy, double oz, double side,
                      int64_t depth, uint64_t* codes, int* bad, void* stream);
/* Stable radix sort of codes (bits [0, end_bit)); perm_out = original indices
 * (the reference's stable argsort). */
int kifmm_tree_sort(const uint64_t* codes_in, int64_t n, int end_bit, uint64_t* codes_out,
                    int64_t* perm_out, void* temp, int64_t temp_bytes, void* stream);
/* Runs of a sorted key array: unique keys, counts, *n_runs (device). */
int kifmm_tree_rle(const uint64_t* keys, int64_t n, uint64_t* unique, int64_t* counts,
                   int64_t* n_runs, void* temp, int64_t temp_bytes, void* stream);
/* Distinct parent codes of a sorted level (*n_out device; scratch: n codes). */
int kifmm_tree_parents(const uint64_t* codes, int64_t n, uint64_t* scratch, uint64_t* parents,
                       int64_t* n_out, void* temp, int64_t temp_bytes, void* stream);
/* Binary search: rows[i] = index of queries[i] in the sorted table or -1. */
int kifmm_lookup_codes(const uint64_t* table, int64_t n, const uint64_t* queries, int64_t nq,
                       int64_t* rows, void* stream);
/* Near-field candidates (engine.py:231-240): rows (ntl, 27), own leaf first,
 * then the in-domain neighbours by ascending code, -1 = absent. */
int kifmm_near_field_rows(const uint64_t* tleaf, int64_t ntl, int64_t depth,
                          const uint64_t* sleaf, int64_t nsl, int64_t* rows, void* stream);
/* BLAS-M2L source table in the sweep layout src[tile][j][m] (n_slots % 128
 * == 0): source row at anchor(slot_target) + offset(class_tv[class][j]). */
int kifmm_blas_src_table(const uint64_t* tcodes, const int32_t* slot_target, int64_t n_slots,
                         int64_t level, const int32_t* class_tv, const int8_t* offsets,
                         const uint64_t* scodes, int64_t ns, int32_t* src, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KIFMM_B200_H */
