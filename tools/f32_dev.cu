// Development timing harness for the FP32 apply kernel (NEXT-3): instantiates one shape of
// kernel_f32.cuh at nbw = 64 and times prep + apply at (n, nev) with CUDA events.  Not a
// parity check (tests/test_gpu_f32.py is); used to compare kernel variants quickly.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSD=2 -DSCW=2 -DSNC=1 \
//        -I paper_1811_01277_b200/csrc -o tools/f32_dev tools/f32_dev.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "kernel_f32.cuh"
using namespace elpa_b200;
#ifndef SD
#define SD 2
#endif
#ifndef SCW
#define SCW 2
#endif
#ifndef SK
#define SK 1
#endif
#ifndef SNC
#define SNC 1
#endif
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__global__ void fill(float *v, float *tau, int64_t R, int b, float *Q, int64_t nq) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t s = 0x9E3779B97F4A7C15ull * (i + 1);
        float nrm = 1.0f;
        v[i * b] = 1.0f;
        for (int k = 1; k < b; k++) {
            s ^= s >> 12; s ^= s << 25; s ^= s >> 27;
            float x = float((s * 2685821657736338717ull) >> 40) / float(1 << 24) * 2.0f - 1.0f;
            v[i * b + k] = x; nrm += x * x;
        }
        tau[i] = 2.0f / nrm;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x)
        Q[i] = float((i * 2654435761ull) % 2001) / 1000.0f - 1.0f;
}

int main(int argc, char **argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 20000, nev = argc > 2 ? atoll(argv[2]) : 20000;
    const int reps = argc > 3 ? atoi(argv[3]) : 3;
    constexpr int B8 = 8, B = 64;
    using Cfg = F32Cfg<B8, SD, SCW, SNC, SK>;
    const int64_t R = hh_total(n, B), M = num_depths(n, B);
    float *v, *tau, *Q, *ws;
    uint64_t *prog;
    const int64_t ldq = (n + 3) / 4 * 4;
    CK(cudaMalloc(&v, R * B * 4)); CK(cudaMalloc(&tau, R * 4)); CK(cudaMalloc(&Q, ldq * nev * 4));
    const int64_t wsb = total_groups(n, B8, M) * f32_blob_floats(B8) * 4;
    CK(cudaMalloc(&ws, wsb));
    fill<<<1184, 256>>>(v, tau, R, B, Q, ldq * nev);
    CK(cudaDeviceSynchronize());
    const int64_t cols = int64_t(SCW) * SNC * 32, nx = (nev + cols - 1) / cols, items = nx * ((M + SD - 1) / SD);
    CK(cudaMalloc(&prog, (items + 1) * 8));
    auto kern = apply_f32_kernel<B8, SD, SCW, SNC, SK>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM)));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::THREADS, Cfg::SMEM));
    int64_t grid = int64_t(per_sm) * 148;
    if (grid > items) grid = items;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int64_t G0 = groups_at_depth(n, B8, 0);
    float best = 1e30f, bestk = 1e30f;
    for (int r = 0; r < reps + 1; r++) {
        cudaEventRecord(e0);
        prep_f32_kernel<B8><<<dim3(unsigned((G0 + 7) / 8), unsigned(M)), 256>>>(n, v, tau, ws);
        cudaEvent_t ek; cudaEventCreate(&ek); cudaEventRecord(ek);
        CK(cudaMemsetAsync(prog, 0, (items + 1) * 8));
        kern<<<unsigned(grid), Cfg::THREADS, Cfg::SMEM>>>(n, nev, ws, Q, ldq, prog, 32);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms, msk; cudaEventElapsedTime(&ms, e0, e1); cudaEventElapsedTime(&msk, ek, e1);
        if (r > 0) { if (ms < best) best = ms; if (msk < bestk) bestk = msk; }
        cudaEventDestroy(ek);
    }
    CK(cudaGetLastError());
    const double fl = 4.0 * B * double(R) * double(nev);   // credited (upper bound of useful) flops
    printf("{\"variant\":\"%s\",\"shape\":[%d,%d,%d,%d],\"n\":%lld,\"nev\":%lld,\"grid\":%lld,\"per_sm\":%d,\"ms\":%.3f,\"apply_ms\":%.3f,\"tflops\":%.3f,\"apply_tflops\":%.3f}\n",
           VARIANT, SD, SCW, SNC, SK, (long long)n, (long long)nev, (long long)grid, per_sm, best, bestk, fl / best / 1e9, fl / bestk / 1e9);
    return 0;
}
