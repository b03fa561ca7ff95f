// Probe: L2 -> shared-memory ingress per SM through cp.async.bulk (the
// path the tensor-memory sweep feeds its stages by).  One CTA per SM; one
// producer thread keeps NS stages of STAGE bytes in flight (CHUNK bytes per
// bulk copy) from an L2-resident 16 MB buffer, one consumer thread waits
// for each stage and releases it.  Reports bytes/clk/SM and the aggregate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o probe_ingress tools/probe_ingress.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t par) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(par)
        : "memory");
}

__global__ void ingress(const unsigned char* src, size_t src_bytes, int ns, int stage, int chunk,
                        int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t full[16], empty[16];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < ns; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long t0 = clock64();
  if (tid == 0) {
    uint32_t off = (uint32_t)blockIdx.x * 7919u * 1024u;
    const uint32_t mask = (uint32_t)(src_bytes / 2 - 1);    // power of two
    for (int g = 0; g < iters; ++g) {
      const int s = g % ns;
      if (g >= ns) wait(&empty[s], ((g / ns) - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                   "r"(stage)
                   : "memory");
      for (int c = 0; c < stage; c += chunk) {
        off = (off + 4096u + 65536u) & mask & ~127u;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sm + s * stage + c)),
            "l"(src + off), "r"(chunk), "r"(smem_u32(&full[s]))
            : "memory");
      }
    }
  } else if (tid == 32) {
    for (int g = 0; g < iters; ++g) {
      const int s = g % ns;
      wait(&full[s], (g / ns) & 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  const size_t bytes = 16u << 20;
  unsigned char* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct C { int ns, stage, chunk; } cs[] = {
      {3, 57344, 28672}, {4, 49152, 24576}, {6, 32768, 16384}, {8, 24576, 12288},
      {3, 57344, 4096},  {12, 16384, 16384}, {2, 57344, 28672}, {6, 32768, 32768},
      {4, 25088, 25088}, {4, 25088, 6272}, {2, 25088, 25088}, {8, 25088, 25088},
  };
  for (auto c : cs) {
    const int iters = 2000;
    for (int rep = 0; rep < 2; ++rep) {
      ingress<<<148, 64, c.ns * c.stage>>>(src, bytes, c.ns, c.stage, c.chunk, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
    }
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const double bpc = (double)c.stage * iters / avg;
    printf("ns %2d stage %6d chunk %6d: %6.1f B/clk/SM, %5.0f clk/stage, %6.2f TB/s at 1.965 GHz x 148\n",
           c.ns, c.stage, c.chunk, bpc, avg / iters, bpc * 148 * 1.965e9 / 1e12);
    fflush(stdout);
  }
  return 0;
}
