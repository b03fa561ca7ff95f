// Pipe-peak probes for the roofline denominators that MEASURED_PEAKS.json
// does not carry (FP32 FFMA, FP64 DFMA, MUFU rsqrt).  Each thread runs 8
// independent dependency chains so the pipe, not latency, is the limit.
#include "common.cuh"

using namespace kifmm;

namespace {

template <typename T>
__global__ void fma_probe(T* out, int iters, T b, T c) {
  T a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = (T)(threadIdx.x + i) * T(1e-3);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = a[i] * b + c;
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void rsqrt_probe(float* out, int iters, float c) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0f + (threadIdx.x + i) * 1e-3f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = rsqrtf(a[i]) + c;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FP64 tensor-core (DMMA) probes: 128 FMAs per thread per iteration.
__global__ void dmma884_probe(double* out, int iters) {
  double c[8][2];
  const double a = 1e-3 * (threadIdx.x & 7), b = 0.999;
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16816_probe(double* out, int iters) {
  double c[2][4];
  const double a = 1e-3 * (threadIdx.x & 7), b = 0.999;
#pragma unroll
  for (int i = 0; i < 2; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
          "{%4,%4,%4,%4,%4,%4,%4,%4}, {%5,%5,%5,%5}, {%0,%1,%2,%3};"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 2; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Packed FP32 (FFMA2, fma.rn.f32x2): 128 FMAs per thread per iteration.
__global__ void ffma2_probe(float* out, int iters) {
  unsigned long long a[4];
  const float2 b2{0.999f, 0.998f}, c2{1e-4f, 2e-4f};
  const unsigned long long b = *reinterpret_cast<const unsigned long long*>(&b2);
  const unsigned long long c = *reinterpret_cast<const unsigned long long*>(&c2);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 v{1e-3f * (threadIdx.x + i), 2e-3f * (threadIdx.x + i)};
    a[i] = *reinterpret_cast<unsigned long long*>(&v);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(b), "l"(c));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 v = *reinterpret_cast<float2*>(&a[i]);
    s += v.x + v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace

extern "C" {

// kind: 0 = FP32 FFMA, 1 = FP64 DFMA, 2 = MUFU rsqrt (FP32), 3 = DMMA m8n8k4,
// 4 = DMMA m16n8k16 (FP64 tensor cores), 5 = packed FP32 FFMA2.  out must hold
// blocks*threads elements of the probe type.  Work per launch:
// blocks*threads*iters*128 operations (an FMA counts as 2 flops).
int kifmm_probe(int kind, int64_t blocks, int64_t threads, int64_t iters, void* out,
                void* stream) {
  if (blocks < 1 || threads < 1 || iters < 1) return KIFMM_EARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (kind == 0)
    fma_probe<float><<<(unsigned)blocks, (unsigned)threads, 0, s>>>((float*)out, (int)iters,
                                                                     0.999f, 1e-4f);
  else if (kind == 1)
    fma_probe<double><<<(unsigned)blocks, (unsigned)threads, 0, s>>>((double*)out, (int)iters,
                                                                      0.999, 1e-4);
  else if (kind == 2)
    rsqrt_probe<<<(unsigned)blocks, (unsigned)threads, 0, s>>>((float*)out, (int)iters, 0.5f);
  else if (kind == 3)
    dmma884_probe<<<(unsigned)blocks, (unsigned)threads, 0, s>>>((double*)out, (int)iters);
  else if (kind == 4)
    dmma16816_probe<<<(unsigned)blocks, (unsigned)threads, 0, s>>>((double*)out, (int)iters);
  else if (kind == 5)
    ffma2_probe<<<(unsigned)blocks, (unsigned)threads, 0, s>>>((float*)out, (int)iters);
  else
    return KIFMM_EARG;
  return launch_status();
}

}  // extern "C"
