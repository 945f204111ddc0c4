// FP64 peak micro-benchmarks for B200 (sm_100a): DFMA (CUDA-core FP64 pipe) and
// DMMA m8n8k4 (FP64 tensor path via mma.sync).  These fix the roofline
// denominators reported by bench.py (MEASURED_PEAKS.json has no FP64 entry).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int CH>
__global__ void dfma_kernel(double* out, double a, double b, int iters) {
  double c[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) c[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) s += c[i];
  if (s == 12345.678) out[0] = s;
}

template<int CH>
__global__ void dmma_kernel(double* out, double a0, double b0, int iters) {
  double acc[CH][2];
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < CH; i++) { acc[i][0] = i; acc[i][1] = -i; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

// latency: one warp, one dependent chain
__global__ void dmma_lat(double* out, long long* cyc, double a, double b, int iters) {
  double c0 = 0, c1 = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (c0 + c1 == 12345.678) out[0] = c0;
}
__global__ void dfma_lat(double* out, long long* cyc, double a, double b, int iters) {
  double c = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) c = fma(c, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (c == 12345.678) out[0] = c;
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
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\":\"%s\",\"cc\":\"%d.%d\",\"sms\":%d,\"l2_bytes\":%d,\"smem_per_sm\":%zu,\"smem_optin\":%zu,\"regs_per_sm\":%d,\"clock_khz\":%d}\n",
         p.name, p.major, p.minor, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerMultiprocessor,
         p.sharedMemPerBlockOptin, p.regsPerMultiprocessor, clk);
  double* out; CK(cudaMalloc(&out, 64)); long long* cyc; CK(cudaMalloc(&cyc, 64));
  const int sms = p.multiProcessorCount;
  const int iters = 1 << 14;
  // DFMA throughput sweeps (blocks/SM x threads)
  for (int bps : {2, 4, 8}) {
    int grid = sms * bps, thr = 256;
    float ms = timeit([&] { dfma_kernel<8><<<grid, thr>>>(out, 1.0000001, 1e-7, iters); }, 5);
    double fl = 2.0 * 8 * iters * (double)grid * thr;
    printf("{\"test\":\"dfma\",\"blocks_per_sm\":%d,\"threads\":%d,\"chains\":8,\"ms\":%.4f,\"tflops\":%.3f}\n", bps, thr, ms, fl / ms / 1e9);
  }
  for (int bps : {1, 2, 4, 8}) {
    int grid = sms * bps, thr = 128;
    float ms = timeit([&] { dmma_kernel<4><<<grid, thr>>>(out, 1.0000001, 1e-7, iters / 4); }, 5);
    double fl = 2.0 * 256 * 4 * (iters / 4) * (double)grid * (thr / 32);
    printf("{\"test\":\"dmma_m8n8k4\",\"blocks_per_sm\":%d,\"threads\":%d,\"chains\":4,\"ms\":%.4f,\"tflops\":%.3f}\n", bps, thr, ms, fl / ms / 1e9);
  }
  for (int bps : {1, 2, 4}) {
    int grid = sms * bps, thr = 256;
    float ms = timeit([&] { dmma_kernel<8><<<grid, thr>>>(out, 1.0000001, 1e-7, iters / 8); }, 5);
    double fl = 2.0 * 256 * 8 * (iters / 8) * (double)grid * (thr / 32);
    printf("{\"test\":\"dmma_m8n8k4\",\"blocks_per_sm\":%d,\"threads\":%d,\"chains\":8,\"ms\":%.4f,\"tflops\":%.3f}\n", bps, thr, ms, fl / ms / 1e9);
  }
  // latencies
  long long hc;
  dmma_lat<<<1, 32>>>(out, cyc, 1.0, 1e-9, 4096); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost));
  printf("{\"test\":\"dmma_latency_cycles\",\"value\":%.2f}\n", hc / 4096.0);
  dfma_lat<<<1, 32>>>(out, cyc, 1.0, 1e-9, 4096); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost));
  printf("{\"test\":\"dfma_latency_cycles\",\"value\":%.2f}\n", hc / 4096.0);
  // single-SM DMMA throughput vs warps (cycles per DMMA per SM)
  for (int w : {1, 2, 4, 8, 16}) {
    float ms = timeit([&] { dmma_kernel<4><<<1, 32 * w>>>(out, 1.0000001, 1e-7, iters / 4); }, 3);
    double n = 4.0 * (iters / 4) * w;
    printf("{\"test\":\"dmma_1sm\",\"warps\":%d,\"ms\":%.4f,\"ns_per_dmma\":%.4f}\n", w, ms, ms * 1e6 / n);
  }
  return 0;
}
