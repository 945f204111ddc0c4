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
// Kernel: CTA tile (WI*WM) x (WJ*WN) x 16, WI x WJ warps, warp tile WM x WN of 8x8 MMA tiles (up
// to 32 independent accumulator chains), a STAGES-deep cp.async ring (16-byte copies where the
// source is 16-byte aligned, 8-byte copies otherwise; zero fill past M, N, K), shared tiles
// stored [row][k] with the 16-byte chunk index XOR-swizzled by row parity so each quarter-warp's
// 16-byte fragment loads hit 8 distinct bank groups.  With beta != 0 the C tile is prefetched
// into L2 at the start and read-modified-written in the epilogue.
// Split-K: S slices of K.  Slice z writes its partial tile to scratch[z]; the last slice to
// finish a tile (per-tile arrival counter) adds the S partials in slice order — deterministic —
// and writes C.  The counters reset themselves.
// (A persistent variant streaming k-tiles across tiles measured slower: 0.82 vs 0.90 of peak at
// 8192^3, 0.68 vs 0.74 at the K = 256 update.)
#pragma once
#include <stdint.h>

namespace elpa_b200 {

namespace gemm {

constexpr int BK = 16;

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
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

// Load rows [r0, r0 + ROWS) x k [k0, k0 + BK) of a K-contiguous operand (element (k, r) at
// P[k + r*ld]) into a shared tile; rows >= R or k >= K read as zero.
template <int ROWS, int THREADS>
__device__ __forceinline__ void load_tile(double *tile, const double *P, int64_t ld, int r0, int R, int k0, int K) {
    static_assert((ROWS * BK / 2) % THREADS == 0, "tile chunks must divide the threads");
#pragma unroll
    for (int u = 0; u < (ROWS * BK / 2) / THREADS; u++) {
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

template <int WI_, int WJ_, int WM_, int WN_, int STAGES_>
struct Cfg {
    static constexpr int WI = WI_, WJ = WJ_, WM = WM_, WN = WN_, STAGES = STAGES_;
    static constexpr int BM = WI * WM, BN = WJ * WN, THREADS = 32 * WI * WJ;
    static constexpr int MT = WM / 8, NT = WN / 8;
    static constexpr size_t SMEM = size_t(STAGES) * (BM + BN) * BK * sizeof(double);
    // CTAs per SM the registers are capped for (register file 64K, shared memory ~227 KB)
    static constexpr int MINB = (THREADS <= 128 && 3 * SMEM <= 220 * 1024 && MT * NT <= 16) ? 3
                              : (THREADS <= 128 && 2 * SMEM <= 220 * 1024) ? 2 : 1;
};

// The configuration the library uses: 64 x 64 tiles, 4 warps of 32 x 32 (16 accumulator chains
// each, 152 registers), 4 stages (64 KB): three CTAs per SM, so the prologue and epilogue of one
// CTA overlap the main loops of the other two.  Measured against 128 x 64 tiles with 64 x 32 warps
// (two CTAs per SM) in tools/gemm_bench.cu (profiles/r02/gemm_configs_r02.jsonl): 0.92 vs 0.91 of
// the DMMA peak at 8192^3, 0.84 vs 0.74 at the K = 256 update with beta, 0.89 vs 0.82 at the
// split-K V^T Q product.
using Main = Cfg<2, 2, 32, 32, 4>;

// grid (tiles_x, tiles_y, S): x = column tile (fastest, so concurrently running CTAs share their
// A rows in L2), y = row tile, z = K slice.
template <class G, bool BETA>
__global__ void __launch_bounds__(G::THREADS, G::MINB)
dgemm_tn_kernel(int M, int N, int K, int k_per_split, double alpha, const double *__restrict__ A, int64_t lda,
                const double *__restrict__ B, int64_t ldb, double beta, double *C, int64_t ldc, double *scratch,
                unsigned *counters, int kmode) {
    constexpr int BM = G::BM, BN = G::BN, STAGES = G::STAGES, MT = G::MT, NT = G::NT, THREADS = G::THREADS;
    extern __shared__ __align__(128) double smem[];
    __shared__ unsigned s_last;
    double *sA = smem;                               // [STAGES][BM * BK]
    double *sB = smem + STAGES * BM * BK;            // [STAGES][BN * BK]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wi = warp / G::WJ, wj = warp % G::WJ;
    const int q = lane & 3, rl = lane >> 2;
    const int i0 = blockIdx.y * BM, j0 = blockIdx.x * BN;
    const int S = gridDim.z;
    const bool direct = (S == 1);                    // no split: this CTA owns the final tile
    int kz0 = blockIdx.z * k_per_split;
    int kz1 = min(K, kz0 + k_per_split);
    // structural zeros the caller declares (kmode, gemm_tn): the tile skips k ranges where its
    // B columns (bit 1: B(k, j) = 0 for k < j) or A rows (bit 2: A(k, i) = 0 for k < i) are zero,
    // or B is upper triangular (bit 4: B(k, j) = 0 for k > j)
    if (kmode & 1) kz0 = max(kz0, j0 & ~(BK - 1));
    if (kmode & 2) kz0 = max(kz0, i0 & ~(BK - 1));
    if (kmode & 4) kz1 = min(kz1, j0 + BN);
    const int nkt = kz1 > kz0 ? (kz1 - kz0 + BK - 1) / BK : 0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; s++) {
        if (s < nkt) {
            load_tile<BM, THREADS>(sA + s * BM * BK, A, lda, i0, M, kz0 + s * BK, kz1);
            load_tile<BN, THREADS>(sB + s * BN * BK, B, ldb, j0, N, kz0 + s * BK, kz1);
        }
        commit();
    }
    if (BETA && direct) {
        // pull the C tile into L2 now, so the epilogue's read-modify-write hits L2
        constexpr int LINES = (BN * 8 + 127) / 128 + 1;
        for (int e = threadIdx.x; e < BM * LINES; e += THREADS) {
            const int r = e / LINES, l = e % LINES;
            const int i = i0 + r;
            if (i >= M) continue;
            const uintptr_t a = (reinterpret_cast<uintptr_t>(C + int64_t(i) * ldc + j0) & ~uintptr_t(127)) +
                                uintptr_t(l) * 128;
            if (a < reinterpret_cast<uintptr_t>(C + int64_t(i) * ldc + min(N, j0 + BN)))
                asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
        }
    }

    double2 acc[MT][NT];
#pragma unroll
    for (int a = 0; a < MT; a++)
#pragma unroll
        for (int b = 0; b < NT; b++) acc[a][b] = make_double2(0.0, 0.0);

    for (int kt = 0; kt < nkt; kt++) {
        wait_group<STAGES - 2>();
        __syncthreads();
        {
            const int kn = kt + STAGES - 1;
            if (kn < nkt) {
                const int st = kn % STAGES;
                load_tile<BM, THREADS>(sA + st * BM * BK, A, lda, i0, M, kz0 + kn * BK, kz1);
                load_tile<BN, THREADS>(sB + st * BN * BK, B, ldb, j0, N, kz0 + kn * BK, kz1);
            }
            commit();
        }
        const double *tA = sA + (kt % STAGES) * BM * BK;
        const double *tB = sB + (kt % STAGES) * BN * BK;
#pragma unroll
        for (int kk = 0; kk < BK / 8; kk++) {
            double2 fa[MT], fb[NT];
#pragma unroll
            for (int a = 0; a < MT; a++)
                fa[a] = *reinterpret_cast<const double2 *>(tA + swz(wi * G::WM + a * 8 + rl, kk * 4 + q));
#pragma unroll
            for (int b = 0; b < NT; b++)
                fb[b] = *reinterpret_cast<const double2 *>(tB + swz(wj * G::WN + b * 8 + rl, kk * 4 + q));
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

    if (direct) {
        // lane holds C[i][j], C[i][j+1], i = .. + lane/4, j = .. + 2(lane%4).  With beta, the NT
        // old values of a row are read together before any store: a store may alias a later load
        // in the compiler's view, so interleaving them would serialise one L2 round trip each
        // (measured: 2x slower at K = 256).
#pragma unroll
        for (int a = 0; a < MT; a++) {
            const int i = i0 + wi * G::WM + a * 8 + rl;
            if (i >= M) continue;
            double *crow = C + int64_t(i) * ldc;
            double2 old[NT];
            bool vec[NT];
#pragma unroll
            for (int b = 0; b < NT; b++) {
                const int j = j0 + wj * G::WN + b * 8 + 2 * q;
                const double *p = crow + j;
                vec[b] = j + 1 < N && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
                old[b] = make_double2(0.0, 0.0);
                if (BETA) {
                    if (vec[b]) old[b] = __ldcg(reinterpret_cast<const double2 *>(p));
                    else {
                        if (j < N) old[b].x = __ldcg(p);
                        if (j + 1 < N) old[b].y = __ldcg(p + 1);
                    }
                }
            }
#pragma unroll
            for (int b = 0; b < NT; b++) {
                const int j = j0 + wj * G::WN + b * 8 + 2 * q;
                if (j >= N) continue;
                double2 v = make_double2(alpha * acc[a][b].x, alpha * acc[a][b].y);
                if (BETA) {
                    v.x = fma(beta, old[b].x, v.x);
                    v.y = fma(beta, old[b].y, v.y);
                }
                double *p = crow + j;
                if (vec[b]) {
                    *reinterpret_cast<double2 *>(p) = v;
                } else {
                    p[0] = v.x;
                    if (j + 1 < N) p[1] = v.y;
                }
            }
        }
        return;
    }

    // split-K: partial tile -> scratch[z] (tile-local layout [BM][BN]); the last arrival sums
    // the slices in order z = 0 .. S-1 and writes C
    const int tile = blockIdx.y * gridDim.x + blockIdx.x;
    const int64_t tsz = int64_t(BM) * BN;
    double *mine = scratch + (int64_t(blockIdx.z) * gridDim.x * gridDim.y + tile) * tsz;
#pragma unroll
    for (int a = 0; a < MT; a++)
#pragma unroll
        for (int b = 0; b < NT; b++) {
            const int il = wi * G::WM + a * 8 + rl, jl = wj * G::WN + b * 8 + 2 * q;
            *reinterpret_cast<double2 *>(mine + il * BN + jl) = acc[a][b];
        }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(counters + tile, 1u);
        s_last = (prev == unsigned(S - 1)) ? 1u : 0u;
        if (s_last) counters[tile] = 0u;             // self-resetting for the next call
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int64_t zs = int64_t(gridDim.x) * gridDim.y * tsz;
    for (int e = threadIdx.x; e < BM * BN / 2; e += THREADS) {
        const int il = (2 * e) / BN, jl = (2 * e) % BN;
        const int i = i0 + il, j = j0 + jl;
        if (i >= M || j >= N) continue;
        const double *src = scratch + int64_t(tile) * tsz + il * BN + jl;
        double2 sum = make_double2(0.0, 0.0);
        for (int z = 0; z < S; z++) {
            const double2 v = __ldcg(reinterpret_cast<const double2 *>(src + z * zs));
            sum.x += v.x;
            sum.y += v.y;
        }
        double *p = C + int64_t(i) * ldc + j;
        double2 v = make_double2(alpha * sum.x, alpha * sum.y);
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

}  // namespace gemm
}  // namespace elpa_b200
