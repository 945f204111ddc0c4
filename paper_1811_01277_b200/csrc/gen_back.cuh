// gen_back.cuh — NEXT-4: the generalized back-transformation
//     V = (L^{-1})^T Vtilde        (Eq. 7; B = L L^T)
// i.e. the triangular solve L^T V = Vtilde for nev columns.  Left-looking blocked form over
// row blocks of kGbBlock from the bottom: for block b (rows [r0, r1)),
//     Q_b <- Q_b - L[r1:n, r0:r1]^T Q[r1:n]      (contraction, k = n - r1)
//     Q_b <- (L_bb^{-1})^T Q_b                    (contraction with the inverted diagonal block)
// This file holds the diagonal-block inversion kernel; the products run in the library's own
// DMMA contraction (dgemm_dmma.cuh), as for NEXT-1.
#pragma once
#include <stdint.h>

namespace elpa_b200 {

constexpr int kGbBlock = 128;

// Inverse of every diagonal block L_bb (m x m, m = min(128, n - 128 b)), one CTA per block:
// the block is staged in shared memory (row-major, 128 KB), thread j computes column j of
// X = L_bb^{-1} by forward substitution, X[i][j] = (delta_ij - sum_{k=j}^{i-1} L[i][k] X[k][j]) / L[i][i],
// writing X column-major (ld 128) to Linv + b*128*128.  Entries above the diagonal are zero.
__global__ void __launch_bounds__(kGbBlock)
gb_trinv_kernel(int64_t n, const double *__restrict__ L, int64_t ldl, double *__restrict__ Linv) {
    constexpr int NB = kGbBlock;
    extern __shared__ double sL[];                       // sL[i * NB + k] = L[r0 + i][r0 + k]
    const int64_t b = blockIdx.x, r0 = b * NB;
    const int m = int((n - r0) < NB ? (n - r0) : NB);
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int k = e / m, i = e % m;                  // column k of L is contiguous in i
        sL[i * NB + k] = (i >= k) ? L[(r0 + k) * ldl + r0 + i] : 0.0;
    }
    __syncthreads();
    const int j = threadIdx.x;
    if (j >= m) return;
    double *x = Linv + b * NB * NB + int64_t(j) * NB;    // column j of X
    for (int i = 0; i < j; i++) x[i] = 0.0;
    for (int i = j; i < m; i++) {
        double s = 0.0;
        for (int k = j; k < i; k++) s = fma(sL[i * NB + k], x[k], s);
        x[i] = ((i == j ? 1.0 : 0.0) - s) / sL[i * NB + i];
    }
}

}  // namespace elpa_b200
