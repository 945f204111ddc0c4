// dgemm_dmma.cuh — the library's own FP64 tensor-core contraction for the dense steps next to
// the hot path: NEXT-1 (band -> full back-transformation: the compact-WY panel
// products) and NEXT-4 (generalized back-transformation, Eq. 7: the blocked
// triangular solve).  One form covers every product those paths need:
//
//     C[i*ldc + j] = alpha * sum_k A[k + i*lda] * B[k + j*ldb]  (+ beta * C[i*ldc + j])
//
// i.e. C (M x N, stored row-major: j contiguous) = alpha * A^T B with A (K x M) and B (K x N)
// column-major, both K-contiguous.  That is the layout the m8n8k4 FP64 MMA wants on both sides:
// a lane holds two consecutive k of one row of A^T and one column of B (the k index of the
// 8-deep step is permuted so lane q takes k = 2q, 2q+1 — the sum is the same, only its order
// changes), and the accumulator gives every lane two consecutive j of one i, stored as one
// 16-byte pair.  Callers choose which matrix is "A" so the output's contiguous index is j.
//
// Kernel: CTA tile 128 x 128 x 16, 8 warps as 2 (i) x 4 (j), warp tile 64 x 32 = 8 x 4 MMA tiles
// (32 independent accumulator chains), a 4-stage cp.async ring (16-byte copies where the source
// is 16-byte aligned, 8-byte copies otherwise; zero fill past M, N, K), shared tiles stored
// [row][k] with the 16-byte chunk index XOR-swizzled by row parity so each quarter-warp's
// 16-byte fragment loads hit 8 distinct bank groups.  Split-K: grid.z slices of K, slice z
// writing its own partial C_z = C + z * split_stride with beta = 0 (deterministic; a reduction
// kernel adds the slices).
#pragma once
#include <stdint.h>

namespace elpa_b200 {

namespace gemm {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4, THREADS = 256;
constexpr int WM = 64, WN = 32;                 // warp tile
constexpr int MT = WM / 8, NT = WN / 8;         // MMA tiles per warp
constexpr size_t SMEM = size_t(STAGES) * (BM + BN) * BK * sizeof(double);   // 128 KB

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16(uint32_t dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp8(uint32_t dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// shared tile [row][BK] doubles, 8 chunks of 16 bytes per row; chunk c of row r lives at
// physical chunk c ^ ((r & 1) << 2)
__device__ __forceinline__ int swz(int r, int c) { return r * BK + 2 * (c ^ ((r & 1) << 2)); }

// Load rows [r0, r0 + 128) x k [k0, k0 + BK) of a K-contiguous operand (element (k, r) at
// P[k + r*ld]) into a shared tile; rows >= R or k >= K read as zero.  4 chunks per thread.
__device__ __forceinline__ void load_tile(double *tile, const double *P, int64_t ld, int r0, int R, int k0, int K) {
#pragma unroll
    for (int u = 0; u < (BM * BK / 2) / THREADS; u++) {
        const int e = threadIdx.x + u * THREADS;
        const int r = e >> 3, c = e & 7;
        const int k = k0 + 2 * c;
        const uint32_t dst = smem_addr(tile + swz(r, c));
        const int row = r0 + r;
        const bool rin = row < R;
        const double *src = P + (rin ? int64_t(row) * ld : 0) + (k < K ? k : 0);
        const int avail = rin ? K - k : 0;               // valid doubles from k on (may be <= 0)
        if ((reinterpret_cast<uintptr_t>(src) & 15) == 0 || avail <= 0) {
            cp16(dst, src, avail >= 2 ? 16u : (avail == 1 ? 8u : 0u));
        } else {                                         // 8-byte aligned only: two copies
            cp8(dst, src, 8u);
            cp8(dst + 8, avail >= 2 ? src + 1 : src, avail >= 2 ? 8u : 0u);
        }
    }
}

template <bool BETA>
__global__ void __launch_bounds__(THREADS, 1)
dgemm_tn_kernel(int M, int N, int K, int k_per_split, double alpha, const double *__restrict__ A, int64_t lda,
                const double *__restrict__ B, int64_t ldb, double beta, double *C, int64_t ldc,
                int64_t split_stride) {
    extern __shared__ __align__(128) double smem[];
    double *sA = smem;                               // [STAGES][BM * BK]
    double *sB = smem + STAGES * BM * BK;            // [STAGES][BN * BK]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wi = warp >> 2, wj = warp & 3;         // 2 x 4 warps
    const int i0 = blockIdx.y * BM, j0 = blockIdx.x * BN;
    const int kz0 = blockIdx.z * k_per_split;
    const int kz1 = min(K, kz0 + k_per_split);
    C += int64_t(blockIdx.z) * split_stride;
    const int nkt = kz1 > kz0 ? (kz1 - kz0 + BK - 1) / BK : 0;

    double2 acc[MT][NT];
#pragma unroll
    for (int a = 0; a < MT; a++)
#pragma unroll
        for (int b = 0; b < NT; b++) acc[a][b] = make_double2(0.0, 0.0);

#pragma unroll
    for (int s = 0; s < STAGES - 1; s++) {
        if (s < nkt) {
            load_tile(sA + s * BM * BK, A, lda, i0, M, kz0 + s * BK, kz1);
            load_tile(sB + s * BN * BK, B, ldb, j0, N, kz0 + s * BK, kz1);
        }
        commit();
    }
    const int q = lane & 3, rl = lane >> 2;
    for (int kt = 0; kt < nkt; kt++) {
        wait_group<STAGES - 2>();
        __syncthreads();
        {
            const int kn = kt + STAGES - 1;
            if (kn < nkt) {
                const int st = kn % STAGES;
                load_tile(sA + st * BM * BK, A, lda, i0, M, kz0 + kn * BK, kz1);
                load_tile(sB + st * BN * BK, B, ldb, j0, N, kz0 + kn * BK, kz1);
            }
            commit();
        }
        const double *tA = sA + (kt % STAGES) * BM * BK;
        const double *tB = sB + (kt % STAGES) * BN * BK;
#pragma unroll
        for (int kk = 0; kk < BK / 8; kk++) {
            double2 fa[MT], fb[NT];
#pragma unroll
            for (int a = 0; a < MT; a++) {
                const int r = wi * WM + a * 8 + rl;
                fa[a] = *reinterpret_cast<const double2 *>(tA + swz(r, kk * 4 + q));
            }
#pragma unroll
            for (int b = 0; b < NT; b++) {
                const int r = wj * WN + b * 8 + rl;
                fb[b] = *reinterpret_cast<const double2 *>(tB + swz(r, kk * 4 + q));
            }
#pragma unroll
            for (int a = 0; a < MT; a++)
#pragma unroll
                for (int b = 0; b < NT; b++) dmma(acc[a][b].x, acc[a][b].y, fa[a].x, fb[b].x);
#pragma unroll
            for (int a = 0; a < MT; a++)
#pragma unroll
                for (int b = 0; b < NT; b++) dmma(acc[a][b].x, acc[a][b].y, fa[a].y, fb[b].y);
        }
    }
    wait_group<0>();

    // epilogue: lane holds C[i][j], C[i][j+1], i = .. + lane/4, j = .. + 2(lane%4)
#pragma unroll
    for (int a = 0; a < MT; a++) {
        const int i = i0 + wi * WM + a * 8 + rl;
        if (i >= M) continue;
        double *crow = C + int64_t(i) * ldc;
#pragma unroll
        for (int b = 0; b < NT; b++) {
            const int j = j0 + wj * WN + b * 8 + 2 * q;
            if (j >= N) continue;
            double2 v = make_double2(alpha * acc[a][b].x, alpha * acc[a][b].y);
            double *p = crow + j;
            if (j + 1 < N && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
                if (BETA) {
                    const double2 o = *reinterpret_cast<const double2 *>(p);
                    v.x = fma(beta, o.x, v.x);
                    v.y = fma(beta, o.y, v.y);
                }
                *reinterpret_cast<double2 *>(p) = v;
            } else {
                if (BETA) v.x = fma(beta, p[0], v.x);
                p[0] = v.x;
                if (j + 1 < N) {
                    if (BETA) v.y = fma(beta, p[1], v.y);
                    p[1] = v.y;
                }
            }
        }
    }
}

// Sum of split-K slices: C[i*ldc + j] = sum_z P[z*zs + i*ldp + j] (+ beta * C[i*ldc + j], and
// + add[i*ldadd + j] when add != nullptr), for i < M, j < N.
__global__ void __launch_bounds__(256)
splitk_reduce_kernel(int M, int N, int S, const double *__restrict__ P, int64_t ldp, int64_t zs, double beta,
                     const double *add, int64_t ldadd, double *C, int64_t ldc) {
    const int64_t total = int64_t(M) * N;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = e / N, j = e % N;
        double s = 0.0;
        for (int z = 0; z < S; z++) s += P[z * zs + i * ldp + j];
        if (add) s += add[i * ldadd + j];
        if (beta != 0.0) s = fma(beta, C[i * ldc + j], s);
        C[i * ldc + j] = s;
    }
}

}  // namespace gemm
}  // namespace elpa_b200
