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

// T factor of every panel from its Gram matrix G_p = V_p^T V_p (P x P, symmetric), LAPACK dlarft
// forward: T[a][a] = tau_a, T[0:a, a] = -tau_a T[0:a, 0:a] G[0:a, a].  T is stored column-major
// (T[a*P + i] = T[i][a]).  Blocked in 64 x 64 blocks (the recurrence for a block column of
// reflectors J given the earlier ones is T[0:J, J] = -T[0:J, 0:J] G[0:J, J] T_JJ, the standard
// two-block form of the compact WY factor):
//   1. T_JJ by the column recurrence above on the diagonal block, in shared memory;
//   2. for every earlier row block I: X = sum_{K = I}^{J-1} T[I, K] G[K, J]  (T is upper
//      triangular), then T[I, J] = -X T_JJ, block products from shared memory.
// One CTA (512 threads) per panel; P must be a multiple of 64.  (The unblocked recurrence read
// T from L2 one dependent load at a time: 14 ms per call at n = 20000, P = 512.)
constexpr int kTB = 64, kTS = 65;                 // block size, padded shared-memory row stride
constexpr size_t kTfactorSmem = size_t(4) * kTB * kTS * sizeof(double);

__global__ void __launch_bounds__(512)
b2f_tfactor(int64_t K, int64_t P, const double *__restrict__ tau, const double *__restrict__ G,
            double *__restrict__ T) {
    extern __shared__ double sm[];
    double *Gd = sm, *Td = sm + kTB * kTS, *Ab = sm + 2 * kTB * kTS, *Bb = sm + 3 * kTB * kTS;
    const int64_t p = blockIdx.x;
    const double *g = G + p * P * P;
    double *t = T + p * P * P;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int r = tid >> 3, c0 = (tid & 7) * 8;     // block products: row r, columns c0 .. c0+7
    const int nb = int(P / kTB);
    for (int64_t e = tid; e < P * P; e += nt) t[e] = 0.0;
    for (int J = 0; J < nb; J++) {
        const int64_t a0 = int64_t(J) * kTB;
        // 1. diagonal block
        for (int e = tid; e < kTB * kTB; e += nt) {
            const int i = e % kTB, k = e / kTB;         // G column-major: G[k][i] at g[k*P + i]
            Gd[i * kTS + k] = g[(a0 + k) * P + a0 + i];
            Td[i * kTS + k] = 0.0;
        }
        __syncthreads();
        for (int a = 0; a < kTB; a++) {
            const double ta = (p * P + a0 + a < K) ? tau[p * P + a0 + a] : 0.0;
            if (tid < a) {
                double s = 0.0;
                for (int k = tid; k < a; k++) s = fma(Td[tid * kTS + k], Gd[k * kTS + a], s);
                Td[tid * kTS + a] = -ta * s;
            }
            if (tid == a) Td[a * kTS + a] = ta;
            __syncthreads();
        }
        for (int e = tid; e < kTB * kTB; e += nt) {
            const int i = e % kTB, k = e / kTB;
            t[(a0 + k) * P + a0 + i] = Td[i * kTS + k];
        }
        // 2. off-diagonal blocks T[I, J], I < J
        for (int I = 0; I < J; I++) {
            double acc[8];
#pragma unroll
            for (int u = 0; u < 8; u++) acc[u] = 0.0;
            for (int Kb = I; Kb < J; Kb++) {
                __syncthreads();
                for (int e = tid; e < kTB * kTB; e += nt) {
                    const int i = e % kTB, k = e / kTB;
                    Ab[i * kTS + k] = __ldcg(t + (int64_t(Kb) * kTB + k) * P + int64_t(I) * kTB + i);   // T[I,Kb]
                    Bb[i * kTS + k] = g[(a0 + k) * P + int64_t(Kb) * kTB + i];                           // G[Kb,J]
                }
                __syncthreads();
                for (int k = 0; k < kTB; k++) {
                    const double av = Ab[r * kTS + k];
#pragma unroll
                    for (int u = 0; u < 8; u++) acc[u] = fma(av, Bb[k * kTS + c0 + u], acc[u]);
                }
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < 8; u++) Ab[r * kTS + c0 + u] = acc[u];      // X
            __syncthreads();
            double out[8];
#pragma unroll
            for (int u = 0; u < 8; u++) out[u] = 0.0;
            for (int k = 0; k < kTB; k++) {
                const double xv = Ab[r * kTS + k];
#pragma unroll
                for (int u = 0; u < 8; u++) out[u] = fma(xv, Td[k * kTS + c0 + u], out[u]);
            }
#pragma unroll
            for (int u = 0; u < 8; u++) t[(a0 + c0 + u) * P + int64_t(I) * kTB + r] = -out[u];
        }
        __syncthreads();
    }
}

}  // namespace elpa_b200
