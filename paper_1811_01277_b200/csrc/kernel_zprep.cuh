// kernel_zprep.cuh — complex reflector preparation (NEXT-3 second half, R15) and the
// complex bring-up kernel.
//
// prep_zmma_kernel: for every group (m, g) of 8 sweeps (geometry.cuh), the window-local complex
// reflector block V_g ((b+8) x 8, column a = sweep 8g+6-a starting at window row 7-a, v_0 = 1),
// the forward compact-WY factor T' of conj(tau) (zlarft: G_0 ... G_7 = I - V T' V^H for
// G_a = H_a^H), U' = -V T', written as m8n8k4 B-fragments of Re U', Im U', Re V, Im V
// (layout of kernel_prep.cuh, one array per part).  One warp per group.
// Complex data are interleaved (re, im) doubles: hh_v is R x nbw complex, hh_tau R complex.
#pragma once
#include "geometry.cuh"

namespace elpa_b200 {

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 zconj(double2 a) { return make_double2(a.x, -a.y); }

template <int B8>
__global__ void __launch_bounds__(64)
prep_zmma_kernel(int64_t n, const double *__restrict__ hh_v, const double *__restrict__ hh_tau,
                 double *__restrict__ blobs) {
    constexpr int B = 8 * B8;
    constexpr int LAM = B8 + 1;
    constexpr int WR = 8 * LAM;
    __shared__ double2 Vs[2][WR][9];
    __shared__ double2 Ts[2][8][8];
    __shared__ double2 Gs[2][8][8];
    __shared__ double2 taus[2][8];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t m = blockIdx.y;
    const int64_t g = (int64_t)blockIdx.x * 2 + warp;
    if (g >= groups_at_depth(n, B8, m)) return;
    double2(*V)[9] = Vs[warp];
    const int64_t Jm = n - 3 - m * B;

    for (int idx = lane; idx < WR * 8; idx += 32) V[idx >> 3][idx & 7] = make_double2(0.0, 0.0);
    if (lane < 8) taus[warp][lane] = make_double2(0.0, 0.0);
    __syncwarp();
    for (int a = 0; a < 8; a++) {
        const int64_t j = 8 * g + 6 - a;
        if (j < 0 || j > Jm) continue;
        const int64_t s = j + 1 + m * B;
        const int64_t L = (n - s < B) ? (n - s) : B;
        const int64_t r = hh_off(j, n, B) + m;
        const double *v = hh_v + 2 * r * B;
        for (int i = lane; i < L; i += 32)
            V[7 - a + i][a] = (i == 0) ? make_double2(1.0, 0.0) : make_double2(v[2 * i], v[2 * i + 1]);
        if (lane == 0) taus[warp][a] = make_double2(hh_tau[2 * r], -hh_tau[2 * r + 1]);   // conj(tau)
    }
    __syncwarp();
    // G = V^H V
    for (int e = lane; e < 64; e += 32) {
        const int p = e >> 3, a = e & 7;
        double2 acc = make_double2(0.0, 0.0);
        for (int w = 0; w < WR; w++) {
            const double2 t = zmul(zconj(V[w][p]), V[w][a]);
            acc.x += t.x;
            acc.y += t.y;
        }
        Gs[warp][p][a] = acc;
    }
    for (int e = lane; e < 64; e += 32) Ts[warp][e >> 3][e & 7] = make_double2(0.0, 0.0);
    __syncwarp();
    // zlarft forward: T'[a][a] = tau'_a; T'[0:a, a] = -tau'_a T'[0:a, 0:a] G[0:a, a]
    for (int a = 0; a < 8; a++) {
        const double2 ta = taus[warp][a];
        double2 t = make_double2(0.0, 0.0);
        if (lane < a) {
            for (int p = lane; p < a; p++) {
                const double2 x = zmul(Ts[warp][lane][p], Gs[warp][p][a]);
                t.x += x.x;
                t.y += x.y;
            }
            t = zmul(make_double2(-ta.x, -ta.y), t);
        }
        __syncwarp();
        if (lane < a) Ts[warp][lane][a] = t;
        if (lane == a) Ts[warp][a][a] = ta;
        __syncwarp();
    }
    double *blob = blobs + (group_base(n, B8, m) + g) * blob_doubles(LAM, 2);
    auto U = [&](int w, int a) {                          // U' = -V T'
        double2 acc = make_double2(0.0, 0.0);
        for (int p = 0; p <= a; p++) {
            const double2 x = zmul(V[w][p], Ts[warp][p][a]);
            acc.x += x.x;
            acc.y += x.y;
        }
        return make_double2(-acc.x, -acc.y);
    };
    const int kq = lane & 3, gq = lane >> 2;
    double2 *dUr = reinterpret_cast<double2 *>(blob);
    double2 *dUi = dUr + 32 * LAM, *uVr = dUr + 64 * LAM, *uVi = dUr + 96 * LAM;
    for (int i = 0; i < LAM; i++) {
        const double2 u0 = U(8 * i + 2 * kq, gq), u1 = U(8 * i + 2 * kq + 1, gq);
        const double2 v0 = V[8 * i + gq][2 * kq], v1 = V[8 * i + gq][2 * kq + 1];
        dUr[i * 32 + lane] = make_double2(u0.x, u1.x);
        dUi[i * 32 + lane] = make_double2(u0.y, u1.y);
        uVr[i * 32 + lane] = make_double2(v0.x, v1.x);
        uVi[i * 32 + lane] = make_double2(v0.y, v1.y);
    }
}

// Complex bring-up kernel: one thread per column, exact reverse generation order, the plain
// complex formulas with explicitly rounded products and sums in the oracle's order
// ((a+bi)(c+di) = (ac - bd) + (ad + bc)i), so the result is bitwise the oracle's
// (oracle.c:oracle_apply_c).  Any nbw.
__global__ void __launch_bounds__(128)
apply_reference_c_kernel(int64_t n, int64_t b, int64_t nev, const double *__restrict__ hh_v,
                         const double *__restrict__ hh_tau, double *Q, int64_t ldq) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nev) return;
    double *q = Q + 2 * c * ldq;
    for (int64_t j = n - 3; j >= 0; j--) {
        const int64_t Mj = (n - 3 - j) / b + 1;
        const int64_t off = hh_off(j, n, b);
        for (int64_t m = Mj - 1; m >= 0; m--) {
            const int64_t r = off + m, s = j + 1 + m * b;
            const int64_t L = (n - s < b) ? (n - s) : b;
            const double *v = hh_v + 2 * r * b;
            double sr = q[2 * s], si = q[2 * s + 1];
            for (int64_t i = 1; i < L; i++) {                // sum += conj(v_i) q_{s+i}
                const double vr = v[2 * i], nvi = -v[2 * i + 1];
                const double qr = q[2 * (s + i)], qi = q[2 * (s + i) + 1];
                sr = __dadd_rn(sr, __dsub_rn(__dmul_rn(vr, qr), __dmul_rn(nvi, qi)));
                si = __dadd_rn(si, __dadd_rn(__dmul_rn(vr, qi), __dmul_rn(nvi, qr)));
            }
            const double tr = hh_tau[2 * r], ti = hh_tau[2 * r + 1];
            const double wr = __dsub_rn(__dmul_rn(tr, sr), __dmul_rn(ti, si));
            const double wi = __dadd_rn(__dmul_rn(tr, si), __dmul_rn(ti, sr));
            q[2 * s] = __dsub_rn(q[2 * s], wr);
            q[2 * s + 1] = __dsub_rn(q[2 * s + 1], wi);
            for (int64_t i = 1; i < L; i++) {                // q_{s+i} -= w v_i
                const double vr = v[2 * i], vi = v[2 * i + 1];
                q[2 * (s + i)] = __dsub_rn(q[2 * (s + i)], __dsub_rn(__dmul_rn(wr, vr), __dmul_rn(wi, vi)));
                q[2 * (s + i) + 1] = __dsub_rn(q[2 * (s + i) + 1], __dadd_rn(__dmul_rn(wr, vi), __dmul_rn(wi, vr)));
            }
        }
    }
}

}  // namespace elpa_b200
