// Probe: throughput of tcgen05.mma kind::tf32 (M = 128, K = 8 per
// instruction) with A in TMEM or in shared memory, for the N shapes of the
// BLAS-M2L sweeps.  One CTA per SM (148 CTAs); one thread issues R rounds of
// 7 fully unrolled k-steps (descriptors precomputed: the issue loop is a few
// uniform-datapath instructions per MMA), each k-step one MMA of N1 columns
// and optionally one of N2 into ND rotating accumulators; clock64 around
// issue + completion.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o probe_mma_rate tools/probe_mma_rate.cu
#include <cstdio>
#include <cstdint>

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
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t db, uint32_t id) {
  asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n" ::"r"(d), "r"(a),
               "l"(db), "r"(id));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t da, uint64_t db, uint32_t id) {
  asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n" ::"r"(d), "l"(da),
               "l"(db), "r"(id));
}

// BG: background work of warps 1..4 while warp 0 issues the MMAs:
// 0 none, 1 tcgen05.st into TMEM, 2 tcgen05.ld from TMEM, 3 LDS.128 from shared memory.
__device__ volatile int g_stop;
// NC: tcgen05.commit (to an unwatched barrier) after every round; DOFF/AOFF: column offsets of D / A.
// WT: after every round, wait on an already-completed mbarrier (1) and fence::after_thread_sync (2)
template <int N1, int N2, bool AT, int ND, int BG = 0, int NC = 0, int DOFF = 0, int AOFF = 384, int WT = 0>
__global__ void rate(int rounds, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2[4];
  __shared__ uint64_t donebar;
  __shared__ uint32_t slot;
  constexpr int KIN = 56;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int i = 0; i < 4; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2[i])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&donebar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&donebar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  __shared__ volatile int stop;
  if (tid == 0) stop = 0;
  __syncthreads();
  if (warp >= 1 && warp <= 4 && BG) {
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    uint32_t v[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    float acc = 0.f;
    int it = 0;
    while (!stop && it < (1 << 22)) {
      ++it;
      if (BG == 1) {
        for (int c = 0; c < 14; ++c)
          asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                           tmem + lane_base + 256 + (c & 7) * 8),
                       "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      } else if (BG == 2) {
        for (int c = 0; c < 14; ++c) {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                         "=r"(v[6]), "=r"(v[7])
                       : "r"(tmem + lane_base + 256 + (c & 7) * 8));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          acc += __uint_as_float(v[0]);
        }
      } else {
        const float4* p = reinterpret_cast<const float4*>(sm + 100 * 1024);
        for (int c = 0; c < 14; ++c) {
          float4 x = p[(tid * 8 + c * 32 + it) & 2047];
          acc += x.x + x.w;
        }
      }
    }
    if (acc == 12345.f) cyc[0] = 0;
  }
  if (tid == 0) {
    constexpr uint32_t id1 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N1 >> 3) << 17) | (8u << 24);
    constexpr uint32_t id2 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N2 >> 3) << 17) | (8u << 24);
    constexpr uint32_t sbo = (KIN / 4) * 128;
    const uint64_t db0 = desc_nosw(smem_u32(sm), 128, sbo);
    const uint64_t da0 = desc_nosw(smem_u32(sm) + 64 * 1024, 128, sbo);
    const uint32_t a0 = tmem + AOFF;
    long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
#pragma unroll
      for (int ks = 0; ks < KIN / 8; ++ks) {
        const uint32_t d = tmem + DOFF + (uint32_t)((ks % ND) * (ND > 1 ? 256 / ND : 0));
        if (AT) {
          mma_ts(d, a0 + ks * 8, db0 + ks * 16, id1);
          if (N2) mma_ts(d, a0 + 64 + ks * 8, db0 + ks * 16, id2);
        } else {
          mma_ss(d, da0 + ks * 16, db0 + ks * 16, id1);
          if (N2) mma_ss(d, da0 + 2048 + ks * 16, db0 + ks * 16, id2);
        }
      }
      if (WT == 1 || WT == 2) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile(
              "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
              "selp.u32 %0, 1, 0, p;\n}\n"
              : "=r"(ok)
              : "r"(smem_u32(&donebar))
              : "memory");
        if (WT == 2) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      } else if (WT == 3) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile(
              "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\n"
              "selp.u32 %0, 1, 0, p;\n}\n"
              : "=r"(ok)
              : "r"(smem_u32(&donebar))
              : "memory");
      } else if (WT == 4) {
        // plain shared-memory flag poll (volatile load)
        volatile int* f = reinterpret_cast<volatile int*>(&bar2[3]);
        while (*f == 12345) {}
      } else if (WT == 5) {
        asm volatile("bar.sync 1, 32;" ::: "memory");
      }
      for (int c = 0; c < NC; ++c)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar2[c]))
                     : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&bar))
                 : "memory");
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
          "selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(smem_u32(&bar))
          : "memory");
    }
    cyc[blockIdx.x] = clock64() - t0;
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N1, int N2, bool AT, int ND, int BG = 0, int NC = 0, int DOFF = 0, int AOFF = 384, int WT = 0>
void run(long long* d) {
  const int rounds = 4000;
  cudaFuncSetAttribute(rate<N1, N2, AT, ND, BG, NC, DOFF, AOFF, WT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  for (int rep = 0; rep < 2; ++rep) {
    rate<N1, N2, AT, ND, BG, NC, DOFF, AOFF, WT><<<148, 160, 160 * 1024>>>(rounds, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return;
    }
  }
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double ksteps = (double)rounds * 7;
  const double flop = 2.0 * 128 * (N1 + N2) * 8 * ksteps;
  printf("WT %d NC %d DOFF %3d AOFF %3d BG %d A %-4s N1 %3d N2 %3d ND %d: %6.1f clk/k-step, %5.0f flop/clk/SM (%5.0f TF/s at 148 SMs x 1.965 GHz)\n",
         WT, NC, DOFF, AOFF, BG, AT ? "tmem" : "smem", N1, N2, ND, avg / ksteps, flop / avg, flop / avg * 148 * 1.965e9 / 1e12);
  fflush(stdout);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  run<112, 64, true, 1>(d);
  run<112, 64, true, 1, 0, 0, 0, 384, 1>(d);
  run<112, 64, true, 1, 0, 0, 0, 384, 3>(d);
  run<112, 64, true, 1, 0, 0, 0, 384, 4>(d);
  run<112, 64, true, 1, 0, 1, 0, 384, 0>(d);
  run<112, 64, true, 1, 0, 1, 0, 384, 3>(d);
  return 0;
}
