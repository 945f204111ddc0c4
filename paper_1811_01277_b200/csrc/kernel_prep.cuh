// kernel_prep.cuh — reflector preparation for the DMMA path.
//
// For every group (m, g) of k = 8 consecutive sweeps at one depth (geometry.cuh), build
// the window-local reflector block V_g ((b+8) x 8, column a = reflector of sweep 8g+6-a,
// starting at window row 7-a, v_0 = 1, zero outside [7-a, 7-a+L)) and the forward compact-WY
// factor T (dlarft, upper triangular: H_0 H_1 ... H_7 = I - V T V^T), and store them as
// ready-to-use m8n8k4 FP64 MMA B-fragments, lane-ordered so each warp reads a group with
// conflict-free 16-byte shared-memory loads, with U = -V T folded in:
//   dotB[i][lane] = (U[8i + 2(lane%4)][lane/4],  U[8i + 2(lane%4) + 1][lane/4])
//   updB[i][lane] = (V[8i + lane/4][2(lane%4)],  V[8i + lane/4][2(lane%4) + 1])
// One warp per group.  Missing reflectors (j < 0 or j > J_m) get tau = 0 (identity).
#pragma once
#include "geometry.cuh"

namespace elpa_b200 {

// Groups [g_lo, g_hi) of every depth (blockIdx.y = depth m): the multi-GPU path prepares the
// groups whose sweeps have arrived while the broadcast of later sweeps is still in flight.
template <int B8, int KIND>
__global__ void __launch_bounds__(128)
prep_dmma_kernel(int64_t n, const double *__restrict__ hh_v, const double *__restrict__ hh_tau,
                 double *__restrict__ blobs, int64_t g_lo, int64_t g_hi) {
    constexpr int B = 8 * B8;
    constexpr int LAM = B8 + 1;
    constexpr int WR = 8 * LAM;                  // window rows
    __shared__ double Vs[4][WR][9];              // +1 pad column
    __shared__ double Ts[4][8][8];
    __shared__ double Gs[4][8][8];
    __shared__ double taus[4][8];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t m = blockIdx.y;
    const int64_t g = g_lo + (int64_t)blockIdx.x * 4 + warp;
    if (g >= g_hi || g >= groups_at_depth(n, B8, m)) return;  // warp-uniform; no block barriers below
    double(*V)[9] = Vs[warp];
    const int64_t Jm = n - 3 - m * B;

    for (int idx = lane; idx < WR * 8; idx += 32) V[idx >> 3][idx & 7] = 0.0;
    // the 8 reflectors' loads are all issued before any is used (one memory latency per group,
    // not eight): lane holds elements lane + 32 u of each vector
    constexpr int PER = (B + 31) / 32;
    double vv[8][PER], tv[8];
    int64_t Ls[8];
#pragma unroll
    for (int a = 0; a < 8; a++) {
        const int64_t j = 8 * g + 6 - a;
        const bool ex = j >= 0 && j <= Jm;
        const int64_t s = j + 1 + m * B;
        Ls[a] = ex ? ((n - s < B) ? (n - s) : B) : 0;
        const int64_t r = ex ? hh_off(j, n, B) + m : 0;
        const double *v = hh_v + r * B;
#pragma unroll
        for (int u = 0; u < PER; u++) {
            const int i = lane + 32 * u;
            vv[a][u] = (i < Ls[a]) ? v[i] : 0.0;
        }
        tv[a] = ex ? hh_tau[r] : 0.0;
    }
    __syncwarp();
#pragma unroll
    for (int a = 0; a < 8; a++) {
#pragma unroll
        for (int u = 0; u < PER; u++) {
            const int i = lane + 32 * u;
            if (i < Ls[a]) V[7 - a + i][a] = (i == 0) ? 1.0 : vv[a][u];
        }
        if (lane == 0) taus[warp][a] = tv[a];
    }
    __syncwarp();
    // Gram matrix G = V^T V on the FP64 tensor cores: 9 chunks x 2 DMMA.8x8x4 (K = window rows,
    // k-pair permuted as in the apply kernel).  Lane (g = lane/4, q = lane%4) supplies rows 2q, 2q+1
    // of the chunk in column g for both operands (A = V^T, B = V hold the same values) and receives
    // G[g][2q], G[g][2q+1].
    const int kq = lane & 3, gq = lane >> 2;
    {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < LAM; i++) {
            const double x0 = V[8 * i + 2 * kq][gq], x1 = V[8 * i + 2 * kq + 1][gq];
            asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(acc.x), "+d"(acc.y) : "d"(x0), "d"(x0));
            asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(acc.x), "+d"(acc.y) : "d"(x1), "d"(x1));
        }
        Gs[warp][gq][2 * kq] = acc.x;
        Gs[warp][gq][2 * kq + 1] = acc.y;
    }
    if (lane < 64 / 2) { Ts[warp][lane >> 3][lane & 7] = 0.0; Ts[warp][(lane + 32) >> 3][(lane + 32) & 7] = 0.0; }
    __syncwarp();
    // dlarft forward: T[a][a] = tau_a; T[0:a, a] = -tau_a * T[0:a, 0:a] * G[0:a, a]
    for (int a = 0; a < 8; a++) {
        double ta = taus[warp][a];
        double t = 0.0;
        if (lane < a) {
            for (int p = lane; p < a; p++) t = fma(Ts[warp][lane][p], Gs[warp][p][a], t);
            t = -ta * t;
        }
        __syncwarp();
        if (lane < a) Ts[warp][lane][a] = t;
        if (lane == a) Ts[warp][a][a] = ta;
        __syncwarp();
    }
    double *blob = blobs + (group_base(n, B8, m) + g) * blob_doubles(LAM, KIND);
    // U^T = -T^T V^T on the tensor cores (M = reflector a, N = window rows in 9 tiles, K = 8
    // reflectors in 2 k-steps): the accumulator of tile i is (U[8i+2q][g], U[8i+2q+1][g]) — the dot
    // B-fragment layout of the apply kernel — and the B operand (V[8i+g][2q], V[8i+g][2q+1]) is the
    // update B-fragment.  (U = -V T: the dot phase then yields W^T = Q_W^T U directly, so the apply
    // kernel needs no separate T step.)
    const double ta0 = -Ts[warp][2 * kq][gq], ta1 = -Ts[warp][2 * kq + 1][gq];
#pragma unroll
    for (int i = 0; i < LAM; i++) {
        double2 d = make_double2(0.0, 0.0), u;
        u.x = V[8 * i + gq][2 * kq];
        u.y = V[8 * i + gq][2 * kq + 1];
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
            : "+d"(d.x), "+d"(d.y) : "d"(ta0), "d"(u.x));
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
            : "+d"(d.x), "+d"(d.y) : "d"(ta1), "d"(u.y));
        reinterpret_cast<double2 *>(blob)[i * 32 + lane] = d;
        reinterpret_cast<double2 *>(blob + 64 * LAM)[i * 32 + lane] = u;
    }
}

}  // namespace elpa_b200
