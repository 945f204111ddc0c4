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

// 16-byte cp.async global -> shared with zero fill of the bytes past `src_bytes` (0, 8, 16)
__device__ __forceinline__ void cp_async16_zfill(void *dst, const void *src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

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
__device__ __forceinline__ void load_pair_async(double2 *dst, const double *Q, int64_t ldq, int64_t n, int64_t col,
                                                bool colok, int64_t r) {
    const bool ok = colok && r >= 0 && r < n;
    const double *src = ok ? Q + col * ldq + r : Q;
    cp_async16_zfill(dst, src, ok ? (r + 1 < n ? 16u : 8u) : 0u);
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

__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(uint64_t *p, uint64_t v) {
    asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int B8, int D, int CW, int NCT>
struct DmmaCfg {
    static constexpr int LAM = B8 + 1;
    static constexpr int BLOB = 128 * LAM + 64;            // doubles per group
    static constexpr int NWARP = D * CW;
    static constexpr int THREADS = 32 * NWARP;
    static constexpr int T = CW * NCT;                     // 8-column tiles per work item
    static constexpr int STAGES = (D * BLOB * 8 * 3 <= 150 * 1024) ? 3 : 2;
    // shared memory: STAGES x D blobs, 2 parities x D x CW x NCT hand-off chunks, barriers
    static constexpr size_t SMEM_BLOBS = size_t(STAGES) * D * BLOB * sizeof(double);
    static constexpr size_t SMEM_HAND = size_t(2) * D * CW * NCT * 64 * sizeof(double);
    static constexpr size_t SMEM_INTAKE = size_t(2) * CW * NCT * 64 * sizeof(double);   // warp-0 HBM intake
    static constexpr size_t SMEM = SMEM_BLOBS + SMEM_HAND + SMEM_INTAKE + 64;
};

// Progress word of work item (x, p): e means pass p of tile group x has
// finalised every chunk >= C0 + 2 - e (kPassDone: the item is complete).  One word per item:
// a word shared by the passes of a tile group would be overwritten by the consumer itself.
constexpr uint64_t kPassDone = ~0ull;

// Persistent kernel: work item k = (pass p = k / NX, tile group x = k % NX) over depth block
// [p*D, p*D + D) and tiles [x*T, x*T + T).  CTAs dequeue items in increasing k from a global
// counter (prog[NX*NP]).  Item (x, p) consumes the rows item (x, p-1) emits, gated by
// prog[k - NX] (release/acquire), so consecutive passes of one tile group pipeline across CTAs.
// Deadlock-free without any co-residency assumption: an item waits only on an item of
// smaller index, which a running CTA dequeued earlier and finishes by induction.
template <int B8, int D, int CW, int NCT>
__global__ void __launch_bounds__(DmmaCfg<B8, D, CW, NCT>::THREADS, 1)
apply_dmma_kernel(int64_t n, int64_t nev, const double *__restrict__ blobs, double *Q, int64_t ldq,
                  uint64_t *prog) {
    using Cfg = DmmaCfg<B8, D, CW, NCT>;
    constexpr int LAM = Cfg::LAM;
    constexpr int BLOB = Cfg::BLOB;
    constexpr int S = Cfg::STAGES;
    constexpr int T = Cfg::T;
    constexpr int64_t B = 8 * B8;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *sblob = reinterpret_cast<double *>(smem_raw);                          // [S][D][BLOB]
    double2 *shand = reinterpret_cast<double2 *>(smem_raw + Cfg::SMEM_BLOBS);      // [2][D][CW][NCT][32]
    double2 *sintake = reinterpret_cast<double2 *>(smem_raw + Cfg::SMEM_BLOBS + Cfg::SMEM_HAND);  // [2][CW][NCT][32]
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + Cfg::SMEM_BLOBS + Cfg::SMEM_HAND + Cfg::SMEM_INTAKE);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int d = warp / CW, cw = warp % CW;
    const int64_t M = num_depths(n, B);
    const int64_t C0 = (n - 2) >> 3;                       // top chunk of every depth's first window
    const int64_t ntile = (nev + 7) >> 3;
    const int64_t NX = (ntile + T - 1) / T;
    const int64_t NP = (M + D - 1) / D;
    const int rsub = 2 * (lane & 3);

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; i++) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    uint32_t phase_bits = 0;  // parity of the next completion, per stage (all threads track it)
    int64_t gstep = 0;        // global step counter (selects the ring stage)
    int64_t *s_item = reinterpret_cast<int64_t *>(bars + S);

    for (;;) {
        if (threadIdx.x == 0)
            *s_item = (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(prog + NX * NP), 1ull);
        __syncthreads();
        const int64_t k = *s_item;
        if (k >= NX * NP) break;
        const int64_t p = k / NX, x = k % NX;
        const int64_t m0 = p * D;
        const int64_t tile_end = min(ntile, (x + 1) * T);
        int64_t col[NCT];
        bool colok[NCT], tileok[NCT];
#pragma unroll
        for (int t = 0; t < NCT; t++) {
            const int64_t tile = x * T + cw * NCT + t;
            tileok[t] = tile < tile_end;
            col[t] = tile * 8 + (lane >> 2);
            colok[t] = tileok[t] && col[t] < nev;
        }
        const int64_t G = groups_at_depth(n, B8, m0);
        const int64_t dmax = min((int64_t)D, M - m0) - 1;
        const int64_t nsteps = G + dmax;
        const int64_t gbase = gstep;

        auto issue = [&](int64_t st) {  // fragments of item step st -> ring stage (gbase+st) % S
            const int64_t gs = gbase + st;
            uint64_t *bar = &bars[gs % S];
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
                    bulk_g2s(sblob + ((gs % S) * D + dd) * BLOB, src, BLOB * 8, bar);
                }
            }
        };
        if (threadIdx.x == 0)
            for (int st = 0; st < S - 1 && st < nsteps; st++) issue(st);

        // cross-pass dependency (warp 0 only): chunk c must be final from pass p-1
        uint64_t seen = 0;
        auto await_chunk = [&](int64_t c) {
            if (p == 0 || c < 0) return;
            const uint64_t need = uint64_t(C0 + 2 - c);
            if (seen >= need) return;
            if (lane == 0) {
                uint64_t v = ld_acquire_u64(prog + (k - NX));
                while (v < need) {
                    __nanosleep(128);
                    v = ld_acquire_u64(prog + (k - NX));
                }
                seen = v;
            }
            seen = __shfl_sync(0xffffffffu, seen, 0);
        };

        double2 q[NCT][LAM];
        if (d == 0) await_chunk(C0);
#pragma unroll
        for (int t = 0; t < NCT; t++)
#pragma unroll
            for (int i = 0; i < LAM; i++)
                q[t][i] = load_pair(Q, ldq, n, col[t], colok[t], 8 * (C0 + d * LAM + i) + rsub);

        // warp 0 streams its new top chunks HBM -> shared (cp.async, 2 slots, one step ahead):
        // the chunk entering at the end of step st is C0 - st - 1, in slot st & 1
        auto intake = [&](int64_t st) {
            const int64_t c = C0 - st - 1;
            await_chunk(c);
#pragma unroll
            for (int t = 0; t < NCT; t++)
                load_pair_async(&sintake[(((st & 1) * CW + cw) * NCT + t) * 32 + lane], Q, ldq, n, col[t], colok[t],
                                8 * c + rsub);
            cp_async_commit();
        };
        if (d == 0) intake(0);
        for (int64_t st = 0; st < nsteps; st++) {
            if (threadIdx.x == 0 && st + S - 1 < nsteps) issue(st + S - 1);
            if (d == 0 && st + 1 < nsteps) intake(st + 1);
            const int64_t g = G - 1 - st + d;
            const bool active = (d <= dmax) && g >= 0 && g < groups_at_depth(n, B8, m0 + d);
            const uint32_t stage = uint32_t((gbase + st) % S);
            const uint32_t par = (phase_bits >> stage) & 1u;
            phase_bits ^= (1u << stage);
            if (active) {
                mbar_wait(&bars[stage], par);
                const double2 *dotB = reinterpret_cast<const double2 *>(sblob + (stage * D + d) * BLOB);
                const double2 *updB = dotB + 32 * LAM;
                const double2 tf = dotB[64 * LAM + lane];
                // Y^T = Q_W^T V_g: independent accumulators per tile (K half x, for NCT = 1,
                // chunk parity) so every warp keeps >= 4 DMMA chains in flight
                constexpr int NACC = (NCT >= 2) ? 2 : 4;
                double2 y[NCT][NACC];
#pragma unroll
                for (int t = 0; t < NCT; t++)
#pragma unroll
                    for (int a = 0; a < NACC; a++) y[t][a] = make_double2(0.0, 0.0);
#pragma unroll
                for (int i = 0; i < LAM; i++) {
                    const double2 vb = dotB[i * 32 + lane];
#pragma unroll
                    for (int t = 0; t < NCT; t++) {
                        if (!tileok[t]) continue;
                        double2 &ya = y[t][(NACC == 4) ? 2 * (i & 1) : 0];
                        double2 &yb = y[t][(NACC == 4) ? 2 * (i & 1) + 1 : 1];
                        dmma(ya.x, ya.y, q[t][i].x, vb.x);
                        dmma(yb.x, yb.y, q[t][i].y, vb.y);
                    }
                }
                // W^T = Y^T (-T)
                double2 w[NCT];
#pragma unroll
                for (int t = 0; t < NCT; t++) {
                    if (!tileok[t]) continue;
                    double ya = y[t][0].x + y[t][1].x, yb = y[t][0].y + y[t][1].y;
                    if (NACC == 4) {
                        ya += y[t][NACC - 2].x + y[t][NACC - 1].x;
                        yb += y[t][NACC - 2].y + y[t][NACC - 1].y;
                    }
                    w[t] = make_double2(0.0, 0.0);
                    dmma(w[t].x, w[t].y, ya, tf.x);
                    dmma(w[t].x, w[t].y, yb, tf.y);
                }
                // Q_W^T += W^T V_g^T
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
            if (st + 1 == nsteps) {       // final windows are written back below
                if (d == 0) cp_async_wait<0>();   // drain the unused last intake before slot reuse
                break;
            }
            const int64_t cbot = C0 - st + d * LAM + LAM - 1;
            if (d == D - 1) {
#pragma unroll
                for (int t = 0; t < NCT; t++) store_pair(Q, ldq, n, col[t], colok[t], 8 * cbot + rsub, q[t][LAM - 1]);
                if ((st & 3) == 3 && cbot <= C0 + 1 && cbot >= 0) {
                    __threadfence();
                    __syncwarp();
                    if (lane == 0) st_release_u64(prog + k, uint64_t(C0 + 2 - cbot));
                }
            } else {
#pragma unroll
                for (int t = 0; t < NCT; t++)
                    shand[((((st & 1) * D + d + 1) * CW + cw) * NCT + t) * 32 + lane] = q[t][LAM - 1];
            }
            if (d == 0) {
                if (st + 1 < nsteps) cp_async_wait<1>(); else cp_async_wait<0>();
            }
            __syncthreads();
#pragma unroll
            for (int t = 0; t < NCT; t++) {
#pragma unroll
                for (int i = LAM - 1; i > 0; i--) q[t][i] = q[t][i - 1];
                if (d == 0) {
                    q[t][0] = sintake[(((st & 1) * CW + cw) * NCT + t) * 32 + lane];
                } else {
                    q[t][0] = shand[((((st & 1) * D + d) * CW + cw) * NCT + t) * 32 + lane];
                }
            }
        }
        // write back the final windows (chunks [C0 - nsteps + 1 + d*LAM, ... + LAM))
#pragma unroll
        for (int t = 0; t < NCT; t++)
#pragma unroll
            for (int i = 0; i < LAM; i++)
                store_pair(Q, ldq, n, col[t], colok[t], 8 * (C0 - (nsteps - 1) + d * LAM + i) + rsub, q[t][i]);
        __threadfence();
        __syncthreads();  // item complete: publish, and the smem ring/hand-off are free again
        if (threadIdx.x == 0) st_release_u64(prog + k, kPassDone);
        gstep += nsteps;
    }
}

}  // namespace elpa_b200
