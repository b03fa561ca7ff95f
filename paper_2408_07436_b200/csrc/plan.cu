// Device tree and plan build (reference octree.py:274-329,
// engine.py:224-256, m2l_blas.py:232-258).  Integer work only, bit-exact with
// the host construction (octree.py / engine.near_field_plan /
// m2l_blas.level_plan_from_buckets), which tests compare it against:
//
//   * encode: Morton code of each point at the leaf level, with the host's
//     float64 arithmetic frac = (p - origin) / side, anchor = min(trunc(frac
//     n), n - 1); code = interleave(x, y, z) << 5 | level;
//   * sort: stable LSD radix sort of (code, point index) pairs (CUB) - the
//     host's stable argsort;
//   * run-length encode of the sorted leaf codes, parent codes + unique for
//     every coarser level (CUB);
//   * lookups: binary search of codes in a level's sorted code array;
//   * near field: per target leaf its own leaf, then the in-domain
//     neighbours in ascending code order, looked up among the source leaves;
//   * BLAS-M2L source table: per tile slot and class vector j, the source
//     row at anchor + offset(class_tv[c][j]) or -1.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_select.cuh>

#include "common.cuh"

using namespace kifmm;

namespace {

constexpr int LEVEL_BITS = 5;
constexpr int kT = 256;

__host__ __device__ __forceinline__ uint64_t spread3(uint64_t x) {
  x &= 0x1fffffull;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}
__host__ __device__ __forceinline__ uint64_t compact3(uint64_t x) {
  x &= 0x1249249249249249ull;
  x = (x ^ (x >> 2)) & 0x10c30c30c30c30c3ull;
  x = (x ^ (x >> 4)) & 0x100f00f00f00f00full;
  x = (x ^ (x >> 8)) & 0x1f0000ff0000ffull;
  x = (x ^ (x >> 16)) & 0x1f00000000ffffull;
  x = (x ^ (x >> 32)) & 0x1fffffull;
  return x;
}
__device__ __forceinline__ uint64_t encode(int64_t ax, int64_t ay, int64_t az, int level) {
  const uint64_t il = (spread3((uint64_t)ax) << 2) | (spread3((uint64_t)ay) << 1) |
                      spread3((uint64_t)az);
  return (il << LEVEL_BITS) | (uint64_t)level;
}
__device__ __forceinline__ void decode(uint64_t code, int64_t& ax, int64_t& ay, int64_t& az) {
  const uint64_t il = code >> LEVEL_BITS;
  ax = (int64_t)compact3(il >> 2);
  ay = (int64_t)compact3(il >> 1);
  az = (int64_t)compact3(il);
}
// Row of `q` in the sorted array `tab` (n entries), -1 if absent.
__device__ __forceinline__ int64_t lookup(const uint64_t* __restrict__ tab, int64_t n, uint64_t q) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(&tab[mid]) < q) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && __ldg(&tab[lo]) == q) ? lo : -1;
}

__global__ void encode_kernel(const double* __restrict__ pts, int64_t n, double ox, double oy,
                              double oz, double side, int depth, uint64_t* __restrict__ codes,
                              int* __restrict__ bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t nb = (int64_t)1 << depth;
  const double o[3] = {ox, oy, oz};
  int64_t a[3];
  bool out = false;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double f = __ddiv_rn(__dsub_rn(pts[i * 3 + d], o[d]), side);
    out |= !(f >= 0.0 && f <= 1.0);
    const int64_t v = (int64_t)__dmul_rn(f, (double)nb);
    a[d] = v < nb - 1 ? v : nb - 1;
  }
  if (out) atomicAdd(bad, 1);
  codes[i] = encode(a[0], a[1], a[2], depth);
}

__global__ void iota_kernel(int64_t* __restrict__ v, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

__global__ void parent_kernel(const uint64_t* __restrict__ codes, int64_t n,
                              uint64_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t c = codes[i];
  const uint64_t level = c & ((1u << LEVEL_BITS) - 1);
  out[i] = (((c >> LEVEL_BITS) >> 3) << LEVEL_BITS) | (level - 1);
}

__global__ void lookup_kernel(const uint64_t* __restrict__ tab, int64_t n,
                              const uint64_t* __restrict__ q, int64_t nq,
                              int64_t* __restrict__ rows) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nq) rows[i] = lookup(tab, n, q[i]);
}

// rows[i*27 + 0] = own leaf among the source leaves, then the in-domain
// neighbours in ascending code order (missing ones -1, in place).
__global__ void near_field_kernel(const uint64_t* __restrict__ tleaf, int64_t ntl, int depth,
                                  const uint64_t* __restrict__ sleaf, int64_t nsl,
                                  int64_t* __restrict__ rows) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntl) return;
  const uint64_t own = tleaf[i];
  int64_t ax, ay, az;
  decode(own, ax, ay, az);
  const int64_t nb = (int64_t)1 << depth;
  uint64_t c[26];
  int m = 0;
  for (int dx = -1; dx <= 1; ++dx)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dz = -1; dz <= 1; ++dz) {
        if (!dx && !dy && !dz) continue;
        const int64_t x = ax + dx, y = ay + dy, z = az + dz;
        if (x < 0 || y < 0 || z < 0 || x >= nb || y >= nb || z >= nb) continue;
        const uint64_t v = encode(x, y, z, depth);
        int k = m++;
        while (k > 0 && c[k - 1] > v) {        // insertion sort, ascending
          c[k] = c[k - 1];
          --k;
        }
        c[k] = v;
      }
  int64_t* r = rows + i * 27;
  r[0] = lookup(sleaf, nsl, own);
  for (int k = 0; k < 26; ++k) r[1 + k] = k < m ? lookup(sleaf, nsl, c[k]) : -1;
}

__global__ void blas_src_kernel(const uint64_t* __restrict__ tcodes,
                                const int32_t* __restrict__ slot_target, int64_t n_slots,
                                int level, const int32_t* __restrict__ class_tv,
                                const int8_t* __restrict__ offsets,
                                const uint64_t* __restrict__ scodes, int64_t ns,
                                int32_t* __restrict__ src) {
  // e walks the device layout [tile][j][m] (slot = tile * 128 + m)
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_slots * 189) return;
  const int64_t tile = e / (189 * 128);
  const int64_t rem = e - tile * (189 * 128);
  const int j = (int)(rem / 128);
  const int64_t slot = tile * 128 + (rem - (int64_t)j * 128);
  const int32_t t = slot_target[slot];
  if (t < 0) {
    src[e] = -1;
    return;
  }
  const uint64_t code = tcodes[t];
  int64_t ax, ay, az;
  decode(code, ax, ay, az);
  const int cls = (int)((code >> LEVEL_BITS) & 7);
  const int tv = class_tv[cls * 189 + j];
  const int64_t x = ax + offsets[3 * tv], y = ay + offsets[3 * tv + 1], z = az + offsets[3 * tv + 2];
  const int64_t nb = (int64_t)1 << level;
  if (x < 0 || y < 0 || z < 0 || x >= nb || y >= nb || z >= nb) {
    src[e] = -1;
    return;
  }
  src[e] = (int32_t)lookup(scodes, ns, encode(x, y, z, level));
}

}  // namespace

extern "C" {

// Scratch bytes of the CUB-backed steps: op 0 = sort (n pairs, key bits
// [0, end_bit)), 1 = run-length encode (n keys), 2 = unique (n keys).  The
// sort's figure includes the index buffer it fills.
int kifmm_tree_temp_bytes(int op, int64_t n, int end_bit, int64_t* bytes) {
  size_t b = 0;
  cudaError_t e = cudaSuccess;
  if (n < 0 || !bytes) return KIFMM_EARG;
  if (op == 0) {
    e = cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                        (const int64_t*)nullptr, (int64_t*)nullptr, n, 0, end_bit);
    b += (((size_t)n * sizeof(int64_t) + 255) / 256) * 256;   // the index buffer, 256-aligned
  } else if (op == 1) {
    e = cub::DeviceRunLengthEncode::Encode(nullptr, b, (const uint64_t*)nullptr,
                                           (uint64_t*)nullptr, (int64_t*)nullptr,
                                           (int64_t*)nullptr, n);
  } else if (op == 2) {
    e = cub::DeviceSelect::Unique(nullptr, b, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (int64_t*)nullptr, n);
  } else {
    return KIFMM_EARG;
  }
  *bytes = (int64_t)b;
  return (int)e;
}

// codes[i] = Morton code of point i (n x 3 float64, row-major) at `depth`;
// *bad (device int, zeroed by the caller) counts points outside the domain.
int kifmm_tree_encode(const double* pts, int64_t n, double ox, double oy, double oz, double side,
                      int64_t depth, uint64_t* codes, int* bad, void* stream) {
  if (n < 0 || depth < 1 || depth > 16 || !(side > 0)) return KIFMM_EARG;
  if (n == 0) return 0;
  encode_kernel<<<ceil_div(n, kT), kT, 0, (cudaStream_t)stream>>>(pts, n, ox, oy, oz, side,
                                                                   (int)depth, codes, bad);
  return launch_status();
}

// Stable sort of codes_in; perm_out[i] = original index of the i-th smallest.
int kifmm_tree_sort(const uint64_t* codes_in, int64_t n, int end_bit, uint64_t* codes_out,
                    int64_t* perm_out, void* temp, int64_t temp_bytes, void* stream) {
  if (n < 0 || end_bit < 1 || end_bit > 64) return KIFMM_EARG;
  if (n == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t* idx = reinterpret_cast<int64_t*>(temp);
  char* cub_temp = reinterpret_cast<char*>(temp) + ((n * sizeof(int64_t) + 255) / 256) * 256;
  size_t cub_bytes = (size_t)temp_bytes - ((n * sizeof(int64_t) + 255) / 256) * 256;
  iota_kernel<<<ceil_div(n, kT), kT, 0, s>>>(idx, n);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(cub_temp, cub_bytes, codes_in, codes_out, idx,
                                                  perm_out, n, 0, end_bit, s);
  return e != cudaSuccess ? (int)e : launch_status();
}

// Runs of equal sorted keys: unique keys, run lengths, *n_runs (device int64).
int kifmm_tree_rle(const uint64_t* keys, int64_t n, uint64_t* unique, int64_t* counts,
                   int64_t* n_runs, void* temp, int64_t temp_bytes, void* stream) {
  if (n < 0) return KIFMM_EARG;
  if (n == 0) return 0;
  size_t b = (size_t)temp_bytes;
  cudaError_t e = cub::DeviceRunLengthEncode::Encode(temp, b, keys, unique, counts, n_runs, n,
                                                     (cudaStream_t)stream);
  return e != cudaSuccess ? (int)e : launch_status();
}

// Sorted distinct parent codes of a sorted level array (*n_out device int64);
// `scratch` holds n codes.
int kifmm_tree_parents(const uint64_t* codes, int64_t n, uint64_t* scratch, uint64_t* parents,
                       int64_t* n_out, void* temp, int64_t temp_bytes, void* stream) {
  if (n < 0) return KIFMM_EARG;
  if (n == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  parent_kernel<<<ceil_div(n, kT), kT, 0, s>>>(codes, n, scratch);
  size_t b = (size_t)temp_bytes;
  cudaError_t e = cub::DeviceSelect::Unique(temp, b, scratch, parents, n_out, n, s);
  return e != cudaSuccess ? (int)e : launch_status();
}

// rows[i] = position of queries[i] in the sorted table, -1 if absent.
int kifmm_lookup_codes(const uint64_t* table, int64_t n, const uint64_t* queries, int64_t nq,
                       int64_t* rows, void* stream) {
  if (n < 0 || nq < 0) return KIFMM_EARG;
  if (nq == 0) return 0;
  lookup_kernel<<<ceil_div(nq, kT), kT, 0, (cudaStream_t)stream>>>(table, n, queries, nq, rows);
  return launch_status();
}

// Near-field candidates (reference engine.py:231-240): rows (ntl, 27) int64,
// own leaf first, then in-domain neighbours by ascending code, -1 = absent.
int kifmm_near_field_rows(const uint64_t* tleaf, int64_t ntl, int64_t depth,
                          const uint64_t* sleaf, int64_t nsl, int64_t* rows, void* stream) {
  if (ntl < 0 || nsl < 0 || depth < 1 || depth > 16) return KIFMM_EARG;
  if (ntl == 0) return 0;
  near_field_kernel<<<ceil_div(ntl, 128), 128, 0, (cudaStream_t)stream>>>(tleaf, ntl, (int)depth,
                                                                          sleaf, nsl, rows);
  return launch_status();
}

// BLAS-M2L source table (m2l_blas.py:232-258 restated per tile slot), in the
// sweep kernels' layout src[tile][j][m] (n_slots a multiple of 128): the
// source row at anchor(target of slot tile*128+m) + offset(class_tv[class][j]).
int kifmm_blas_src_table(const uint64_t* tcodes, const int32_t* slot_target, int64_t n_slots,
                         int64_t level, const int32_t* class_tv, const int8_t* offsets,
                         const uint64_t* scodes, int64_t ns, int32_t* src, void* stream) {
  if (n_slots < 0 || n_slots % 128 || ns < 0 || level < 1 || level > 16) return KIFMM_EARG;
  if (n_slots == 0) return 0;
  const int64_t total = n_slots * 189;
  blas_src_kernel<<<ceil_div(total, kT), kT, 0, (cudaStream_t)stream>>>(
      tcodes, slot_target, n_slots, (int)level, class_tv, offsets, scodes, ns, src);
  return launch_status();
}

}  // extern "C"
