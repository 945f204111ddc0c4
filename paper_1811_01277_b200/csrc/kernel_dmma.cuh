// kernel_dmma.cuh — the hot path: k = 8 compact-WY
// reflector groups applied on FP64 tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4),
// depth-pipelined row windows held in registers.
//
// Work decomposition
//   * A CTA owns a stripe of `tiles_per_cta` 8-column tiles of Q and processes every chase
//     depth for it: passes over depth blocks [m0, m0+D), D depth-warps per column warp.
//   * Warp (d, cw) holds, for its NCT tiles, the b+8-row window of depth m0+d in registers
//     in the m8n8k4 accumulator layout: lane l owns rows 8i + 2(l%4) + {0,1} of column l/4
//     of every 8-row chunk i (lambda = b/8 + 1 chunks, 2 doubles per chunk per tile).
//   * Time step t: warp d applies group g = G_{m0} - 1 - t + d of depth m0+d (sweeps
//     8g+6 .. 8g-1).  The D windows are stacked without overlap (depth m0+d+1 trails depth
//     m0+d by one group, DESIGN.md §5 "schedule legality"); every step they all move up by
//     one 8-row chunk: warp 0 takes the next chunk from HBM, warp d>0 takes the chunk warp
//     d-1 emitted (shared-memory hand-off), warp D-1's emitted chunk goes back to HBM.
//     Each Q row therefore crosses HBM once per D depths.
//   * Per group and tile (all on DMMA):
//        Y^T  = Q_W^T V_g              2*lambda MMAs (K = rows)          [dot products, a4]
//        W^T  = Y^T (-T)               2 MMAs        (K = reflectors)    [recurrence,   a5]
//        Q_W^T += W^T V_g^T            2*lambda MMAs (K = reflectors)    [rank-8 update, a6]
//     The accumulator layout of each product is directly the A-operand layout of the next
//     (K index permuted to match), so no shuffles are needed anywhere.
//   * Prepared fragments of the D groups of the next step are fetched with cp.async.bulk
//     into a 2-stage shared-memory ring completed on an mbarrier (one elected thread).
#pragma once
#include "geometry.cuh"

namespace elpa_b200 {

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Q chunk I/O: lane owns rows r, r+1 (r = 8*chunk + 2*(lane%4)) of column `col`.
__device__ __forceinline__ double2 load_pair(const double *Q, int64_t ldq, int64_t n, int64_t col,
                                             bool colok, int64_t r) {
    double2 v = make_double2(0.0, 0.0);
    if (colok && r >= 0 && r < n) {
        const double *p = Q + col * ldq + r;
        if (r + 1 < n) {
            v = *reinterpret_cast<const double2 *>(p);
        } else {
            v.x = p[0];
        }
    }
    return v;
}
__device__ __forceinline__ void store_pair(double *Q, int64_t ldq, int64_t n, int64_t col, bool colok,
                                           int64_t r, double2 v) {
    if (colok && r >= 0 && r < n) {
        double *p = Q + col * ldq + r;
        if (r + 1 < n) {
            *reinterpret_cast<double2 *>(p) = v;
        } else {
            p[0] = v.x;
        }
    }
}

template <int B8, int D, int CW, int NCT>
struct DmmaCfg {
    static constexpr int LAM = B8 + 1;
    static constexpr int BLOB = 128 * LAM + 64;            // doubles per group
    static constexpr int NWARP = D * CW;
    static constexpr int THREADS = 32 * NWARP;
    // shared memory: 2 stages x D blobs, 2 parities x D x CW x NCT hand-off chunks
    static constexpr size_t SMEM_BLOBS = size_t(2) * D * BLOB * sizeof(double);
    static constexpr size_t SMEM_HAND = size_t(2) * D * CW * NCT * 64 * sizeof(double);
    static constexpr size_t SMEM = SMEM_BLOBS + SMEM_HAND + 64;
};

template <int B8, int D, int CW, int NCT>
__global__ void __launch_bounds__(DmmaCfg<B8, D, CW, NCT>::THREADS, 1)
apply_dmma_kernel(int64_t n, int64_t nev, const double *__restrict__ blobs, double *Q, int64_t ldq,
                  int tiles_per_cta) {
    using Cfg = DmmaCfg<B8, D, CW, NCT>;
    constexpr int LAM = Cfg::LAM;
    constexpr int BLOB = Cfg::BLOB;
    constexpr int64_t B = 8 * B8;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *sblob = reinterpret_cast<double *>(smem_raw);                          // [2][D][BLOB]
    double2 *shand = reinterpret_cast<double2 *>(smem_raw + Cfg::SMEM_BLOBS);      // [2][D][CW][NCT][32]
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + Cfg::SMEM_BLOBS + Cfg::SMEM_HAND);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int d = warp / CW, cw = warp % CW;
    const int64_t M = num_depths(n, B);
    const int64_t C0 = (n - 2) >> 3;                       // top chunk of every depth's first window
    const int64_t ntile = (nev + 7) >> 3;
    const int64_t tile_begin = (int64_t)blockIdx.x * tiles_per_cta;
    const int64_t tile_end = min(ntile, tile_begin + tiles_per_cta);

    int64_t col[NCT];
    bool colok[NCT], tileok[NCT];
#pragma unroll
    for (int t = 0; t < NCT; t++) {
        const int64_t tile = tile_begin + cw * NCT + t;
        tileok[t] = tile < tile_end;
        col[t] = tile * 8 + (lane >> 2);
        colok[t] = tileok[t] && col[t] < nev;
    }
    const int rsub = 2 * (lane & 3);

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    uint32_t phase_bits = 0;  // parity of the next completion, per stage (used by all threads)

    for (int64_t m0 = 0; m0 < M; m0 += D) {
        const int64_t G = groups_at_depth(n, B8, m0);      // groups of depth m0
        const int64_t dmax = min((int64_t)D, M - m0) - 1;  // deepest existing depth in this pass
        const int64_t nsteps = G + dmax;

        // producer: prefetch the fragments of step `st` into stage st&1
        auto issue = [&](int64_t st) {
            uint64_t *bar = &bars[st & 1];
            uint32_t bytes = 0;
            for (int dd = 0; dd <= dmax; dd++) {
                const int64_t g = G - 1 - st + dd;
                if (g >= 0 && g < groups_at_depth(n, B8, m0 + dd)) bytes += BLOB * 8;
            }
            mbar_arrive_expect_tx(bar, bytes);
            for (int dd = 0; dd <= dmax; dd++) {
                const int64_t g = G - 1 - st + dd;
                if (g >= 0 && g < groups_at_depth(n, B8, m0 + dd)) {
                    const double *src = blobs + (group_base(n, B8, m0 + dd) + g) * BLOB;
                    bulk_g2s(sblob + ((st & 1) * D + dd) * BLOB, src, BLOB * 8, bar);
                }
            }
        };
        if (threadIdx.x == 0) issue(0);

        // initial windows: chunks [C0 + d*LAM, C0 + (d+1)*LAM) (only real rows are loaded)
        double2 q[NCT][LAM];
#pragma unroll
        for (int t = 0; t < NCT; t++)
#pragma unroll
            for (int i = 0; i < LAM; i++)
                q[t][i] = load_pair(Q, ldq, n, col[t], colok[t], 8 * (C0 + d * LAM + i) + rsub);

        double2 nxt[NCT];  // warp 0's prefetched next top chunk
        for (int64_t st = 0; st < nsteps; st++) {
            if (threadIdx.x == 0 && st + 1 < nsteps) issue(st + 1);
            if (d == 0) {
#pragma unroll
                for (int t = 0; t < NCT; t++)
                    nxt[t] = load_pair(Q, ldq, n, col[t], colok[t], 8 * (C0 - st - 1) + rsub);
            }
            const int64_t md = m0 + d;
            const int64_t g = G - 1 - st + d;
            const bool active = (d <= dmax) && g >= 0 && g < groups_at_depth(n, B8, md);
            const uint32_t stage = st & 1;
            const uint32_t par = (phase_bits >> stage) & 1u;
            phase_bits ^= (1u << stage);
            if (active) {
                mbar_wait(&bars[stage], par);
                const double2 *dotB = reinterpret_cast<const double2 *>(sblob + (stage * D + d) * BLOB);
                const double2 *updB = dotB + 32 * LAM;
                const double2 tf = dotB[64 * LAM + lane];
                double2 y0[NCT], y1[NCT];
#pragma unroll
                for (int t = 0; t < NCT; t++) { y0[t] = make_double2(0.0, 0.0); y1[t] = make_double2(0.0, 0.0); }
#pragma unroll
                for (int i = 0; i < LAM; i++) {
                    const double2 vb = dotB[i * 32 + lane];
#pragma unroll
                    for (int t = 0; t < NCT; t++) {
                        if (!tileok[t]) continue;
                        if (i & 1) { dmma(y1[t].x, y1[t].y, q[t][i].x, vb.x); dmma(y1[t].x, y1[t].y, q[t][i].y, vb.y); }
                        else       { dmma(y0[t].x, y0[t].y, q[t][i].x, vb.x); dmma(y0[t].x, y0[t].y, q[t][i].y, vb.y); }
                    }
                }
                double2 w[NCT];
#pragma unroll
                for (int t = 0; t < NCT; t++) {
                    if (!tileok[t]) continue;
                    const double ya = y0[t].x + y1[t].x, yb = y0[t].y + y1[t].y;
                    w[t] = make_double2(0.0, 0.0);
                    dmma(w[t].x, w[t].y, ya, tf.x);
                    dmma(w[t].x, w[t].y, yb, tf.y);
                }
#pragma unroll
                for (int i = 0; i < LAM; i++) {
                    const double2 ub = updB[i * 32 + lane];
#pragma unroll
                    for (int t = 0; t < NCT; t++) {
                        if (!tileok[t]) continue;
                        dmma(q[t][i].x, q[t][i].y, w[t].x, ub.x);
                        dmma(q[t][i].x, q[t][i].y, w[t].y, ub.y);
                    }
                }
            }
            if (st + 1 == nsteps) break;  // final windows are written back below
            // emit the bottom chunk
            const int64_t cbot = C0 - st + d * LAM + LAM - 1;
            if (d == D - 1) {
#pragma unroll
                for (int t = 0; t < NCT; t++) store_pair(Q, ldq, n, col[t], colok[t], 8 * cbot + rsub, q[t][LAM - 1]);
            } else {
#pragma unroll
                for (int t = 0; t < NCT; t++)
                    shand[((((st & 1) * D + d + 1) * CW + cw) * NCT + t) * 32 + lane] = q[t][LAM - 1];
            }
            __syncthreads();
            // shift the window down one chunk and take the new top chunk
#pragma unroll
            for (int t = 0; t < NCT; t++) {
#pragma unroll
                for (int i = LAM - 1; i > 0; i--) q[t][i] = q[t][i - 1];
                q[t][0] = (d == 0) ? nxt[t] : shand[((((st & 1) * D + d) * CW + cw) * NCT + t) * 32 + lane];
            }
        }
        // write back the final windows (chunks [C0 - nsteps + 1 + d*LAM, ... + LAM))
#pragma unroll
        for (int t = 0; t < NCT; t++)
#pragma unroll
            for (int i = 0; i < LAM; i++)
                store_pair(Q, ldq, n, col[t], colok[t], 8 * (C0 - (nsteps - 1) + d * LAM + i) + rsub, q[t][i]);
        __syncthreads();  // this pass's stores precede the next pass's loads
    }
}

}  // namespace elpa_b200
