// Probe: tcgen05.mma kind::tf32 with the A operand in TMEM (lane = row,
// column = K element), B in shared memory (K-major, no swizzle).
// D[128 x N] = A[128 x K] . B[N x K]^T, checked against a host product.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o probe_tmem_a tools/probe_tmem_a.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int M = 128;
constexpr int K = 56;
constexpr int N = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc_nosw(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__global__ void probe(const float* A, const float* Bp, float* D, int mode) {
  __shared__ __align__(1024) float sB[N * K];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < N * K; i += blockDim.x) sB[i] = Bp[i];
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  // A into TMEM columns [128, 128 + K): thread tid writes row tid
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  for (int c = 0; c < K; c += 8) {
    uint32_t v[8];
    for (int i = 0; i < 8; ++i) v[i] = __float_as_uint(A[tid * K + c + i]);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     tmem + lane_base + 128 + c),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(M >> 4) << 24);
    const uint32_t sbo = (K / 4) * 128;
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint64_t db = desc_nosw(smem_u32(sB) + ks * 256, 128, sbo);
      const uint32_t acc = ks > 0;
      const uint32_t a_addr = tmem + 128 + ks * (mode == 0 ? 8 : 4);
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
          "r"(a_addr), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&bar))
                 : "memory");
  }
  // wait
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
          "selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(smem_u32(&bar))
          : "memory");
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + lane_base + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) D[tid * N + c + i] = __uint_as_float(v[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  std::vector<float> A(M * K), B(N * K), Bp(N * K), D(M * N);
  srand(1);
  // small integers: exact in tf32 and in the fp32 accumulator
  for (auto& x : A) x = (float)(rand() % 7 - 3);
  for (auto& x : B) x = (float)(rand() % 5 - 2);
  // pack B [n][k] into the canonical no-swizzle K-major layout [n/8][k/4][n%8][k%4]
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k)
      Bp[(((n / 8) * (K / 4) + k / 4) * 8 + n % 8) * 4 + k % 4] = B[n * K + k];
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, Bp.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bp.data(), Bp.size() * 4, cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: error %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
        maxerr = fmax(maxerr, fabs(s - D[m * N + n]));
      }
    printf("mode %d (A column step per k-step = %d): max abs err %g (D[0][0]=%g)\n", mode,
           mode == 0 ? 8 : 4, maxerr, D[0]);
  }
  return 0;
}
