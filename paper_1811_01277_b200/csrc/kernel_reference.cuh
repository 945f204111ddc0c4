// kernel_reference.cuh — bring-up kernel: one thread per eigenvector column,
// reflectors applied in exact reverse generation order (j descending, m descending) with
// explicitly rounded products and sums (no FMA contraction), so the result is bitwise
// equal to the CPU oracle's plain definition (R3, R10).  Correctness anchor for
// the fast kernels; not a performance path.
#pragma once
#include "geometry.cuh"

namespace elpa_b200 {

__global__ void __launch_bounds__(128)
apply_reference_kernel(int64_t n, int64_t b, int64_t nev, const double *__restrict__ hh_v,
                       const double *__restrict__ hh_tau, double *Q, int64_t ldq) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nev) return;
    double *q = Q + c * ldq;
    for (int64_t j = n - 3; j >= 0; j--) {
        int64_t Mj = (n - 3 - j) / b + 1;
        int64_t off = hh_off(j, n, b);
        for (int64_t m = Mj - 1; m >= 0; m--) {
            int64_t r = off + m;
            int64_t s = j + 1 + m * b;
            int64_t L = (n - s < b) ? (n - s) : b;
            const double *v = hh_v + r * b;
            double sum = q[s];                                   // v[0] == 1
            for (int64_t i = 1; i < L; i++) sum = __dadd_rn(sum, __dmul_rn(v[i], q[s + i]));
            double w = __dmul_rn(hh_tau[r], sum);
            q[s] = __dsub_rn(q[s], w);
            for (int64_t i = 1; i < L; i++) q[s + i] = __dsub_rn(q[s + i], __dmul_rn(w, v[i]));
        }
    }
}

}  // namespace elpa_b200
