// dgemm_host.h — launch logic of the library's DMMA contraction (dgemm_dmma.cuh): the split-K
// choice and the scratch it needs.  Used by elpa_b200_dense.cu (NEXT-1, NEXT-4).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "dgemm_dmma.cuh"
#include "host_common.h"

namespace elpa_b200_host {

using GemmCfg = elpa_b200::gemm::Main;

// Split count for C = A^T B with an M x N output and reduction length K.  A small output (the
// V^T Q and L^T Q products have N = 128..256) has a few waves of tiles or fewer, so K is split
// into S slices; S minimises (waves) x (k-steps per slice) plus the partial-sum traffic, in
// seconds at the kernel's per-CTA rate.
inline int gemm_split(int64_t M, int64_t N, int64_t K) {
    using elpa_b200::gemm::BK;
    const int64_t tiles = ((M + GemmCfg::BM - 1) / GemmCfg::BM) * ((N + GemmCfg::BN - 1) / GemmCfg::BN);
    const int64_t slots = int64_t(GemmCfg::MINB) * sm_count();           // resident CTAs
    const int64_t ksteps = (K + BK - 1) / BK;
    const double step_s = 2.0 * GemmCfg::BM * GemmCfg::BN * BK / (36.9e12 / double(slots));
    double best = 1e300;
    int bs = 1;
    for (int S = 1; S <= 16; S++) {
        const int64_t per = (ksteps + S - 1) / S;
        if (S > 1 && per < 8) break;
        const int64_t waves = (tiles * S + slots - 1) / slots;
        const double t = double(waves) * double(per) * step_s + (S > 1 ? double(S + 1) * M * N * 8 / 6e12 : 0.0);
        if (t < best * 0.97) { best = t; bs = S; }
    }
    // Skinny outputs (under two waves of tiles) measured faster with more, power-of-two slices
    // than this model predicts: at M = 20000, N = 128 (the NEXT-4 block products) S = 4-8 reaches
    // 0.88-0.90 of peak for K >= 5000 where the model chose S = 2 (0.83-0.84), and S = 3, 5, 6, 7
    // lose to 4 and 8 (profiles/r02/gemm_split_sweep_n128_r02.jsonl).  So the split is at least
    // the power of two nearest ksteps / 80, capped at 8; and a split the model chose is rounded up
    // to a power of two (at M = 2000, N = 128, K = 19800: S = 13 0.71, S = 16 0.77 of peak;
    // profiles/r02/gemm_split_sweep_small_r02.jsonl).
    if (tiles < 2 * slots) {
        int se = 1;
        while (se < 8 && double(ksteps) / 80.0 >= 1.5 * se) se *= 2;
        bs = std::max(bs, se);
        int p2 = 1;
        while (p2 < bs && p2 < 16) p2 *= 2;
        while (p2 > 1 && ksteps / p2 < 8) p2 /= 2;
        bs = p2;
    }
    return bs;
}

inline int64_t gemm_tiles(int64_t M, int64_t N) {
    return ((M + GemmCfg::BM - 1) / GemmCfg::BM) * ((N + GemmCfg::BN - 1) / GemmCfg::BN);
}

// doubles of split-K scratch one call needs (0 without a split)
inline int64_t gemm_scratch_doubles(int64_t M, int64_t N, int64_t K) {
    const int S = gemm_split(M, N, K);
    return S > 1 ? int64_t(S) * gemm_tiles(M, N) * GemmCfg::BM * GemmCfg::BN : 0;
}

// C (row-major, ldc) = alpha * A^T B (+ beta * C): A (K x M), B (K x N) column-major.
// `scratch` holds gemm_scratch_doubles(M, N, K) doubles; `counters` gemm_tiles(M, N) unsigned
// zero-initialised words (they are left zero again).  alpha must be nonzero.
// kmode declares structural zeros the tiles may skip (the compact-WY panels' staircase):
// GEMM_B_STAIR B(k, j) = 0 for k < j; GEMM_A_STAIR A(k, i) = 0 for k < i; GEMM_B_UPPER
// B(k, j) = 0 for k > j.  The skipped products are exact zeros, so results are unchanged.
enum { GEMM_B_STAIR = 1, GEMM_A_STAIR = 2, GEMM_B_UPPER = 4 };
inline int gemm_tn(int64_t M, int64_t N, int64_t K, double alpha, const double *A, int64_t lda, const double *B,
                   int64_t ldb, double beta, double *C, int64_t ldc, double *scratch, unsigned *counters,
                   cudaStream_t s, int kmode = 0) {
    using namespace elpa_b200::gemm;
    if (M <= 0 || N <= 0) return ELPA_B200_OK;
    if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX || alpha == 0.0) return ELPA_B200_ERR_ARG;
    static bool attr = [] {
        cudaFuncSetAttribute(dgemm_tn_kernel<GemmCfg, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(GemmCfg::SMEM));
        cudaFuncSetAttribute(dgemm_tn_kernel<GemmCfg, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(GemmCfg::SMEM));
        return cudaGetLastError() == cudaSuccess;
    }();
    if (!attr) return ELPA_B200_ERR_CUDA;
    const int S = K > 0 ? gemm_split(M, N, K) : 1;
    const int64_t kps = K > 0 ? ((K + S - 1) / S + BK - 1) / BK * BK : 0;
    const int tx = int((N + GemmCfg::BN - 1) / GemmCfg::BN), ty = int((M + GemmCfg::BM - 1) / GemmCfg::BM);
    const dim3 grid{unsigned(tx), unsigned(ty), unsigned(S)};
    if (beta != 0.0)
        dgemm_tn_kernel<GemmCfg, true><<<grid, GemmCfg::THREADS, GemmCfg::SMEM, s>>>(
            int(M), int(N), int(K), int(kps), alpha, A, lda, B, ldb, beta, C, ldc, scratch, counters, kmode);
    else
        dgemm_tn_kernel<GemmCfg, false><<<grid, GemmCfg::THREADS, GemmCfg::SMEM, s>>>(
            int(M), int(N), int(K), int(kps), alpha, A, lda, B, ldb, 0.0, C, ldc, scratch, counters, kmode);
    return cudaGetLastError() == cudaSuccess ? ELPA_B200_OK : ELPA_B200_ERR_CUDA;
}

}  // namespace elpa_b200_host
