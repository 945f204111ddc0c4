// gemm_bench.cu — development benchmark of the library's DMMA contraction (csrc/dgemm_dmma.cuh)
// in several tile configurations and at the shapes NEXT-1 / NEXT-4 use; checks each against a
// naive FP64 kernel on a ragged small shape first.  Prints one JSON line per (config, shape).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/gemm_bench tools/gemm_bench.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <vector>

#include "../paper_1811_01277_b200/csrc/dgemm_dmma.cuh"

using namespace elpa_b200::gemm;

__global__ void init_kernel(double *p, int64_t n, uint64_t seed) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        uint64_t z = seed + uint64_t(i + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        p[i] = 2.0 * double(z >> 11) * 0x1.0p-53 - 1.0;
    }
}

__global__ void naive_kernel(int M, int N, int K, double alpha, const double *A, int64_t lda, const double *B,
                             int64_t ldb, double beta, double *C, int64_t ldc) {
    const int i = blockIdx.y * 16 + threadIdx.y, j = blockIdx.x * 16 + threadIdx.x;
    if (i >= M || j >= N) return;
    double s = 0.0;
    for (int k = 0; k < K; k++) s += A[k + int64_t(i) * lda] * B[k + int64_t(j) * ldb];
    C[int64_t(i) * ldc + j] = alpha * s + beta * C[int64_t(i) * ldc + j];
}

template <class G>
void run(const char *name, int M, int N, int K, int S, double beta, int reps, bool check) {
    const int64_t lda = K + (K & 1) + 2, ldb = K + (K & 1), ldc = N + 3;
    double *A, *B, *C, *C2, *scr;
    unsigned *cnt;
    const int64_t tiles = int64_t((M + G::BM - 1) / G::BM) * ((N + G::BN - 1) / G::BN);
    cudaMalloc(&A, sizeof(double) * lda * M);
    cudaMalloc(&B, sizeof(double) * ldb * N);
    cudaMalloc(&C, sizeof(double) * ldc * M);
    cudaMalloc(&C2, sizeof(double) * ldc * M);
    cudaMalloc(&scr, sizeof(double) * (S > 1 ? S * tiles * G::BM * G::BN : 1));
    cudaMalloc(&cnt, sizeof(unsigned) * tiles);
    cudaMemset(cnt, 0, sizeof(unsigned) * tiles);
    init_kernel<<<1024, 256>>>(A, lda * M, 1);
    init_kernel<<<1024, 256>>>(B, ldb * N, 2);
    init_kernel<<<1024, 256>>>(C, ldc * M, 3);
    cudaMemcpy(C2, C, sizeof(double) * ldc * M, cudaMemcpyDeviceToDevice);
    cudaFuncSetAttribute(dgemm_tn_kernel<G, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(G::SMEM));
    cudaFuncSetAttribute(dgemm_tn_kernel<G, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(G::SMEM));
    const int64_t kps = ((K + S - 1) / S + BK - 1) / BK * BK;
    const int tx = (N + G::BN - 1) / G::BN, ty = (M + G::BM - 1) / G::BM;
    const dim3 grid(tx, ty, S);
    auto launch = [&](double *c) {
        if (beta != 0.0)
            dgemm_tn_kernel<G, true><<<grid, G::THREADS, G::SMEM>>>(M, N, K, int(kps), -1.0, A, lda, B, ldb, beta, c,
                                                                    ldc, scr, cnt, 0);
        else
            dgemm_tn_kernel<G, false><<<grid, G::THREADS, G::SMEM>>>(M, N, K, int(kps), -1.0, A, lda, B, ldb, 0.0, c,
                                                                     ldc, scr, cnt, 0);
    };
    double err = -1;
    if (check) {
        launch(C);
        naive_kernel<<<dim3((N + 15) / 16, (M + 15) / 16), dim3(16, 16)>>>(M, N, K, -1.0, A, lda, B, ldb, beta, C2, ldc);
        std::vector<double> h1(ldc * M), h2(ldc * M);
        cudaMemcpy(h1.data(), C, sizeof(double) * ldc * M, cudaMemcpyDeviceToHost);
        cudaMemcpy(h2.data(), C2, sizeof(double) * ldc * M, cudaMemcpyDeviceToHost);
        double mx = 0, den = 0;
        for (int64_t i = 0; i < M; i++)
            for (int64_t j = 0; j < ldc; j++) {
                const double a = h1[i * ldc + j], b = h2[i * ldc + j];
                if (j >= N) { if (a != b) mx = 1e300; continue; }
                mx = fmax(mx, fabs(a - b));
                den = fmax(den, fabs(b));
            }
        err = mx / den;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch(C);
    float best = 1e30f;
    for (int r = 0; r < reps; r++) {
        cudaEventRecord(e0);
        launch(C);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = fminf(best, ms);
    }
    const double tf = 2.0 * M * N * double(K) / (best * 1e-3) / 1e12;
    printf("{\"cfg\": \"%s\", \"M\": %d, \"N\": %d, \"K\": %d, \"S\": %d, \"beta\": %g, \"ms\": %.4f, \"tflops\": %.3f, "
           "\"frac\": %.4f, \"err\": %.3g, \"cuda\": \"%s\"}\n",
           name, M, N, K, S, beta, best, tf, tf / 36.983, err, cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
    cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(C2); cudaFree(scr); cudaFree(cnt);
}

template <class G>
void suite(const char *name) {
    run<G>(name, 301, 203, 517, 1, 1.0, 1, true);
    run<G>(name, 301, 203, 517, 3, 0.5, 1, true);
    run<G>(name, 300, 130, 1000, 5, 0.0, 1, true);
    run<G>(name, 8192, 8192, 8192, 1, 0.0, 3, false);
    run<G>(name, 20000, 20000, 256, 1, 1.0, 3, false);     // NEXT-1 Q update
    run<G>(name, 20000, 256, 20000, 1, 0.0, 3, false);     // NEXT-1 W (no split)
    run<G>(name, 20000, 256, 20000, 3, 0.0, 3, false);     // NEXT-1 W (split 3)
    run<G>(name, 20000, 128, 10000, 1, 1.0, 3, false);     // NEXT-4 off-diagonal update
    run<G>(name, 20000, 128, 10000, 4, 1.0, 3, false);
    run<G>(name, 20000, 20000, 512, 1, 1.0, 3, false);     // NEXT-1 Q update, panel 512
    run<G>(name, 20000, 512, 20000, 2, 0.0, 3, false);     // NEXT-1 W, panel 512
}

int main(int argc, char **argv) {
    if (argc >= 6) {      // one shape of the main config: M N K S beta [reps]
        run<Main>("main", atoi(argv[1]), atoi(argv[2]), atoi(argv[3]), atoi(argv[4]), atof(argv[5]),
                  argc > 6 ? atoi(argv[6]) : 3, false);
        return 0;
    }
    if (argc == 2) {      // shape sweep of the main config around the short-K case
        int shapes[][5] = {{20000, 20000, 256, 1, 1}, {20000, 20000, 256, 1, 0}, {8192, 8192, 256, 1, 0},
                           {20000, 20000, 1024, 1, 1}, {20000, 20000, 512, 1, 0}, {8192, 8192, 2048, 1, 0},
                           {20000, 256, 20000, 3, 0}, {20000, 256, 20000, 6, 0}, {20000, 128, 10000, 4, 1},
                           {20000, 128, 10000, 8, 1}, {20000, 20000, 512, 1, 1}};
        for (auto &sh : shapes) run<Main>("main", sh[0], sh[1], sh[2], sh[3], sh[4], 3, false);
        return 0;
    }
    suite<Cfg<2, 2, 64, 32, 4>>("2x2w64x32s4");
    suite<Cfg<2, 2, 64, 32, 3>>("2x2w64x32s3");
    suite<Cfg<2, 2, 32, 32, 4>>("2x2w32x32s4");
    suite<Cfg<2, 2, 32, 32, 3>>("2x2w32x32s3");
    return 0;
}
