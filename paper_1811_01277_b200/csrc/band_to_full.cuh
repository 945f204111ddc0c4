// band_to_full.cuh — NEXT-1: the band -> full eigenvector back-transformation,
// the second of the two transforms every eigenvector goes through in the two-stage solver
// (PAPER.md P:144-146).  Stage-1 reflector j (j = 0 .. K-1, K = n - nbw - 1) acts on rows
// [j + nbw, n) (one reflector per eliminated column of the full -> band reduction):
//      Q <- H_0 H_1 ... H_{K-1} Q.
// Blocked compact WY: panels of P consecutive reflectors, B_p = H_{j0} ... H_{j1-1} =
// I - V_p T_p V_p^T (forward dlarft), applied last panel first as
//      Q <- Q + U_p (V_p^T Q),   U_p = -V_p T_p,
// with the library's DMMA contraction (dgemm_dmma.cuh).  This file holds the panel geometry and
// the preparation kernels (clean panels in both layouts, T factors).
//
// Panel p covers reflectors [p*P, min(K, (p+1)*P)) and rows [r0', n), r0' = (p*P + nbw) & ~1:
// the row origin is rounded down to even so every column segment the contraction streams is
// 16-byte aligned in an even-ldq Q (a leading zero row when p*P + nbw is odd contributes
// nothing).  m_p = n - r0' rows, stored with an even leading dimension ld_p = m_p + (m_p & 1).
#pragma once
#include <stdint.h>

namespace elpa_b200 {

__host__ __device__ inline int64_t b2f_origin(int64_t nbw, int64_t P, int64_t p) { return (p * P + nbw) & ~int64_t(1); }
__host__ __device__ inline int64_t b2f_rows(int64_t n, int64_t nbw, int64_t P, int64_t p) {
    return n - b2f_origin(nbw, P, p);
}
__host__ __device__ inline int64_t b2f_ld(int64_t n, int64_t nbw, int64_t P, int64_t p) {
    const int64_t m = b2f_rows(n, nbw, P, p);
    return m + (m & 1);
}
// offset (doubles) of panel p's V block (ld_p x P, column-major)
__host__ __device__ inline int64_t b2f_panel_offset(int64_t n, int64_t nbw, int64_t P, int64_t p) {
    int64_t off = 0;
    for (int64_t q = 0; q < p; q++) off += b2f_ld(n, nbw, P, q) * P;
    return off;
}

// Clean copy of the panels, column-major: element (i, a) (row r0' + i, reflector j0 + a) is 0
// above the reflector's start row j0 + a + nbw, 1 at it (the implicit v_0), V[j0+a][row] below;
// missing reflectors of the last panel and the padding row are zero.
__global__ void __launch_bounds__(256)
b2f_build_panels(int64_t n, int64_t nbw, int64_t K, int64_t P, const double *__restrict__ V, int64_t ldv,
                 double *__restrict__ Vp) {
    const int64_t p = blockIdx.y;
    const int64_t j0 = p * P;
    const int64_t r0 = b2f_origin(nbw, P, p);
    const int64_t m = b2f_rows(n, nbw, P, p), ld = b2f_ld(n, nbw, P, p);
    double *out = Vp + b2f_panel_offset(n, nbw, P, p);
    const int64_t total = ld * P;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t a = e / ld, i = e % ld;
        const int64_t row = r0 + i, start = j0 + a + nbw;
        double v = 0.0;
        if (j0 + a < K && i < m) {
            if (row == start) v = 1.0;
            else if (row > start) v = V[(j0 + a) * ldv + row];
        }
        out[e] = v;
    }
}

// Row-major copy of one panel (VT[a + i*P] = V_p[i][a]): the K-contiguous operand of U_p = -V_p T_p.
__global__ void __launch_bounds__(256)
b2f_transpose_panel(int64_t m, int64_t ld, int64_t P, const double *__restrict__ Vp, double *__restrict__ VT) {
    __shared__ double tile[32][33];
    const int64_t i0 = int64_t(blockIdx.x) * 32, a0 = int64_t(blockIdx.y) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;    // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = i0 + tx, a = a0 + r;
        tile[r][tx] = (i < m && a < P) ? Vp[a * ld + i] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int64_t i = i0 + r, a = a0 + tx;
        if (i < m && a < P) VT[i * P + a] = tile[tx][r];
    }
}

// T factor of every panel from its Gram matrix G_p = V_p^T V_p (P x P, symmetric):
// T[a][a] = tau_a, T[0:a, a] = -tau_a T[0:a, 0:a] G[0:a, a]  (LAPACK dlarft, forward), T stored
// column-major (T[a*P + i] = T[i][a]).  One CTA per panel; the column recurrence is sequential.
__global__ void __launch_bounds__(256)
b2f_tfactor(int64_t K, int64_t P, const double *__restrict__ tau, const double *__restrict__ G,
            double *__restrict__ T) {
    const int64_t p = blockIdx.x;
    const double *g = G + p * P * P;
    double *t = T + p * P * P;
    for (int64_t e = threadIdx.x; e < P * P; e += blockDim.x) t[e] = 0.0;
    __syncthreads();
    for (int64_t a = 0; a < P; a++) {
        const double ta = (p * P + a < K) ? tau[p * P + a] : 0.0;
        for (int64_t i = threadIdx.x; i < a; i += blockDim.x) {
            double acc = 0.0;
            for (int64_t k = i; k < a; k++) acc = fma(t[k * P + i], g[a * P + k], acc);
            t[a * P + i] = -ta * acc;      // reads column a-1 and earlier only
        }
        if (threadIdx.x == 0) t[a * P + a] = ta;
        __syncthreads();
    }
}

}  // namespace elpa_b200
