// band_to_full.cuh — NEXT-1: the band -> full eigenvector back-transformation,
// the second of the two transforms every eigenvector goes through in the two-stage solver
// (PAPER.md P:144-146).  Stage-1 reflector j (j = 0 .. K-1, K = n - nbw - 1) acts on rows
// [j + nbw, n) (one reflector per eliminated column of the full -> band reduction):
//      Q <- H_0 H_1 ... H_{K-1} Q.
// Blocked compact WY: panels of P consecutive reflectors, B_p = H_{j0} ... H_{j1-1} =
// I - V_p T_p V_p^T (forward dlarft), applied last panel first as Q <- Q - V_p (T_p (V_p^T Q)).
// This file holds the preparation kernels (clean panels, T factors); the three products per
// panel are plain DGEMMs (FP64 tensor cores through cuBLAS, loaded at run time).
#pragma once
#include <stdint.h>

namespace elpa_b200 {

// Panel p covers reflectors [p*P, min(K, (p+1)*P)) and rows [p*P + nbw, n) (m_p rows).
__host__ __device__ inline int64_t b2f_rows(int64_t n, int64_t nbw, int64_t P, int64_t p) {
    return n - (p * P + nbw);
}
// offset (doubles) of panel p's clean V block (m_p x P, column-major, ld = m_p)
__host__ __device__ inline int64_t b2f_panel_offset(int64_t n, int64_t nbw, int64_t P, int64_t p) {
    // sum_{q<p} (n - nbw - q*P) * P
    return P * (p * (n - nbw) - P * p * (p - 1) / 2);
}

// Clean copy of the panels: element (i, a) of panel p is 0 above the reflector's start
// (i < a), 1 at it (i == a, the implicit v_0), V[j0+a][row] below; missing reflectors of the
// last panel are zero columns.
__global__ void __launch_bounds__(256)
b2f_build_panels(int64_t n, int64_t nbw, int64_t K, int64_t P, const double *__restrict__ V, int64_t ldv,
                 double *__restrict__ Vp) {
    const int64_t p = blockIdx.y;
    const int64_t j0 = p * P;
    const int64_t m = b2f_rows(n, nbw, P, p);
    double *out = Vp + b2f_panel_offset(n, nbw, P, p);
    const int64_t total = m * P;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t a = e / m, i = e % m;
        double v = 0.0;
        if (j0 + a < K) {
            if (i == a) v = 1.0;
            else if (i > a) v = V[(j0 + a) * ldv + (j0 + nbw + i)];
        }
        out[e] = v;
    }
}

// T factor of every panel from its Gram matrix G_p = V_p^T V_p (P x P, column-major):
// T[a][a] = tau_a, T[0:a, a] = -tau_a T[0:a, 0:a] G[0:a, a]  (LAPACK dlarft, forward).
// One CTA per panel, thread i owns row i of T; the column recurrence is sequential.
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
