// FP32 peak micro-benchmarks for B200 (sm_100a), for the NEXT-3 FP32 variant's roofline:
// FFMA with all-register operands (the form the apply kernel issues), and the packed
// fma.rn.f32x2 (two FP32 FMAs per lane per instruction, sm_100+).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp32_peak tools/fp32_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

// c[i] = x[i] * y + c[i], x and y live in registers (the apply kernel's q * v + acc shape)
template<int CH>
__global__ void ffma_kernel(float* out, float a, int iters) {
  float c[CH], x[CH];
  float y = a + threadIdx.x * 1e-7f;
#pragma unroll
  for (int i = 0; i < CH; i++) { c[i] = threadIdx.x * 1e-3f + i; x[i] = 1.0f - i * 1e-4f - threadIdx.x * 1e-8f; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) c[i] = fmaf(x[i], y, c[i]);
    y = -y;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) s += c[i];
  if (s == 12345.678f) out[0] = s;
}

__device__ __forceinline__ void ffma2(uint64_t &c, uint64_t a, uint64_t b) {
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(a), "l"(b));
}
template<int CH>
__global__ void ffma2_kernel(float* out, float a, int iters) {
  uint64_t c[CH], x[CH];
  float yv = a + threadIdx.x * 1e-7f;
  uint64_t y;
#pragma unroll
  for (int i = 0; i < CH; i++) {
    float lo = threadIdx.x * 1e-3f + i, hi = -lo;
    c[i] = (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
    float xl = 1.0f - i * 1e-4f, xh = 1.0f + i * 1e-4f;
    x[i] = (uint64_t)__float_as_uint(xl) | ((uint64_t)__float_as_uint(xh) << 32);
  }
  y = (uint64_t)__float_as_uint(yv) | ((uint64_t)__float_as_uint(yv) << 32);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) ffma2(c[i], x[i], y);
    y ^= 0x8000000080000000ull;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) s += __uint_as_float((uint32_t)c[i]) + __uint_as_float((uint32_t)(c[i] >> 32));
  if (s == 12345.678f) out[0] = s;
}

// the apply kernel's dot shape: acc_{k&1} += q_k * v_k with distinct pair registers q_k, v_k
// (three distinct 64-bit operands per FFMA2), 4 accumulators
template<int NQ>
__global__ void ffma2_dot_kernel(float* out, float a, int iters) {
  uint64_t q[NQ], v[NQ], acc[4] = {0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < NQ; i++) {
    float x = a + i * 1e-3f + threadIdx.x * 1e-7f;
    q[i] = (uint64_t)__float_as_uint(x) | ((uint64_t)__float_as_uint(-x) << 32);
    v[i] = (uint64_t)__float_as_uint(0.5f - i * 1e-4f) | ((uint64_t)__float_as_uint(0.25f) << 32);
  }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NQ; i++) ffma2(acc[i & 3], q[i], v[i]);
#pragma unroll
    for (int i = 0; i < NQ; i++) q[i] ^= 0x8000000000000000ull;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) s += __uint_as_float((uint32_t)acc[i]);
  if (s == 12345.678f) out[0] = s;
}

template<typename K>
float timeit(K launch, int reps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  float *out; CK(cudaMalloc(&out, 64));
  const int sms = p.multiProcessorCount, iters = 4096;
  for (int bps : {2, 4, 8}) {
    const int threads = 256, blocks = sms * bps;
    float ms = timeit([&] { ffma_kernel<16><<<blocks, threads>>>(out, 0.999f, iters); }, 5);
    double fl = 2.0 * blocks * threads * 16.0 * iters;
    printf("{\"test\":\"ffma_reg\",\"blocks_per_sm\":%d,\"threads\":%d,\"chains\":16,\"ms\":%.4f,\"tflops\":%.3f}\n",
           bps, threads, ms, fl / ms / 1e9);
    ms = timeit([&] { ffma2_kernel<16><<<blocks, threads>>>(out, 0.999f, iters); }, 5);
    fl = 4.0 * blocks * threads * 16.0 * iters;
    printf("{\"test\":\"ffma2_f32x2\",\"blocks_per_sm\":%d,\"threads\":%d,\"chains\":16,\"ms\":%.4f,\"tflops\":%.3f}\n",
           bps, threads, ms, fl / ms / 1e9);
  }
  for (int bps : {2, 3, 4}) {
    const int threads = 128, blocks = sms * bps;
    float ms = timeit([&] { ffma2_dot_kernel<32><<<blocks, threads>>>(out, 0.999f, iters); }, 5);
    double fl = 4.0 * blocks * threads * 32.0 * iters;
    printf("{\"test\":\"ffma2_dot_3operand\",\"blocks_per_sm\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n",
           bps, threads, ms, fl / ms / 1e9);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
