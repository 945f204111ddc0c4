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
    // Gram matrix G = V^T V (64 entries, 2 per lane)
    for (int e = lane; e < 64; e += 32) {
        const int a = e >> 3, l = e & 7;
        double acc = 0.0;
        for (int w = 0; w < WR; w++) acc = fma(V[w][a], V[w][l], acc);
        Gs[warp][a][l] = acc;
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
    // U = -V T (window rows x 8): the dot phase then yields W^T = Q_W^T U directly
    // (W = -T^T V^T Q_W), so the apply kernel needs no separate T step
    auto U = [&](int w, int a) {
        double acc = 0.0;
        for (int p = 0; p <= a; p++) acc = fma(V[w][p], Ts[warp][p][a], acc);
        return -acc;
    };
    const int kq = lane & 3, gq = lane >> 2;
    for (int i = 0; i < LAM; i++) {
        double2 d, u;
        d.x = U(8 * i + 2 * kq, gq);
        d.y = U(8 * i + 2 * kq + 1, gq);
        u.x = V[8 * i + gq][2 * kq];
        u.y = V[8 * i + gq][2 * kq + 1];
        reinterpret_cast<double2 *>(blob)[i * 32 + lane] = d;
        reinterpret_cast<double2 *>(blob + 64 * LAM)[i * 32 + lane] = u;
    }
}

}  // namespace elpa_b200
