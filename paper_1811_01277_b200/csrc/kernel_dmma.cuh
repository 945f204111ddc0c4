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
//   * Per group and tile (all on DMMA), with U = -V_g T prepared by the prep kernel:
//        W^T  = Q_W^T U                2*lambda MMAs (K = rows)   [dot products + recurrence, a4/a5]
//        Q_W^T += W^T V_g^T            2*lambda MMAs (K = reflectors)           [rank-8 update, a6]
//     The dot accumulator layout is directly the update's A-operand layout (K index permuted
//     to match), so no shuffles are needed anywhere.
//   * Prepared fragments of the D groups of a step are fetched ahead with cp.async.bulk into
//     a 2-3 stage shared-memory ring completed on mbarriers, issued by one thread of the last
//     warp (warp 0 already carries the HBM intake, the item dequeue and the progress publish).
//   * Interior chunks (inside the matrix, every column valid) take a load/store fast path
//     without bounds logic; only the first/last chunks and the last tile group pay for it.
//   * KIND_ZMMA runs complex Hermitian tiles (NEXT-3) as (Re, Im) real tile pairs.  The FP64
//     CUDA-core alternative is a separate kernel (kernel_dfma.cuh).
#pragma once
#include <type_traits>

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
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// Watchdog (debug builds only: ELPA_B200_DEBUG=1 at build time defines ELPA_B200_WATCHDOG): a
// wait longer than ~10 s of wall time (%globaltimer, which is consistent across SMs, unlike
// clock64) is a protocol bug; trap instead of hanging the GPU.  Release builds spin: a trap is a
// sticky error that would poison the caller's whole context, and time-slicing or preemption can
// stretch a correct wait arbitrarily.  No printf: a call inside the wait loops would force the
// live register window across an ABI call boundary.
#ifdef ELPA_B200_WATCHDOG
constexpr unsigned long long kWatchdogNs = 10000000000ull;
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void watchdog_fire() { asm volatile("trap;"); }
#define ELPA_WATCHDOG_START() const unsigned long long elpa_wd_t0 = globaltimer_ns()
#define ELPA_WATCHDOG_CHECK() \
    do { if (globaltimer_ns() - elpa_wd_t0 > kWatchdogNs) watchdog_fire(); } while (0)
#else
#define ELPA_WATCHDOG_START() do { } while (0)
#define ELPA_WATCHDOG_CHECK() do { } while (0)
#endif
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    if (mbar_try_wait(bar, parity)) return;
    ELPA_WATCHDOG_START();
    while (!mbar_try_wait(bar, parity)) ELPA_WATCHDOG_CHECK();
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

// Q chunk I/O: lane owns rows r, r+1 (r = 8*chunk + 2*(lane%4)) of the column starting at
// `colp`; rows outside [0, n) and masked-off columns read as zero and are never written.
__device__ __forceinline__ double2 load_pair(const double *colp, bool ok, int n, int r) {
    double2 v = make_double2(0.0, 0.0);
    if (ok && r >= 0 && r < n) {
        if (r + 1 < n) v = *reinterpret_cast<const double2 *>(colp + r);
        else v.x = colp[r];
    }
    return v;
}
__device__ __forceinline__ void load_pair_async(double2 *dst, const double *colp, bool ok, int n, int r) {
    const bool in = ok && r >= 0 && r < n;
    cp_async16_zfill(dst, in ? colp + r : colp, in ? (r + 1 < n ? 16u : 8u) : 0u);
}
__device__ __forceinline__ void store_pair(double *colp, bool ok, int n, int r, double2 v) {
    if (ok && r >= 0 && r < n) {
        if (r + 1 < n) *reinterpret_cast<double2 *>(colp + r) = v;
        else colp[r] = v.x;
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

// ---------------------------------------------------------------------------------------
// Per-group arithmetic for one warp: its NCT 8-column tiles, window
// q[t][i] in the m8n8k4 accumulator layout (lane l: rows 8i + 2(l%4) + {0,1} of column l/4).
// Two policies compute the same compact-WY group, Q_W <- Q_W - V_g T^T V_g^T Q_W:
// ---------------------------------------------------------------------------------------
enum { KIND_DMMA = 0, KIND_ZMMA = 2 };

// FP64 tensor cores: 2*LAM + 2*LAM DMMA.8x8x4 per tile, no shuffles.  Blob layout (prep
// kernel): dot B-fragments of U = -V_g T [LAM][32 lanes][2], update B-fragments of V_g
// [LAM][32][2] (== V_g row-major 8 x 8 per chunk).
template <int LAM, int NCT>
struct DmmaGroup {
    static constexpr int BLOB = 128 * LAM;
    // tilemask is ignored: a tile past the end of Q holds zeros (masked loads) and is never
    // stored, so computing it costs nothing but keeps every DMMA unpredicated (a predicated
    // mma.sync needs WARPSYNC + NOP padding around it)
    __device__ __forceinline__ static void apply(double2 (&q)[NCT][LAM], const double *blob, uint32_t,
                                                 int lane) {
        const double2 *dotB = reinterpret_cast<const double2 *>(blob);
        const double2 *updB = dotB + 32 * LAM;
        // W^T = Q_W^T U (= -(T^T V_g^T Q_W)^T).  With NCT >= 2 one accumulator chain per tile
        // (the tiles interleave, so consecutive dependent DMMAs are >= NCT issues apart and no
        // DADD combine sits between the phases); NCT = 1 splits the K halves into 2 chains.
        constexpr int NACC = (NCT >= 2) ? 1 : 2;
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
                double2 &ya = y[t][0];
                double2 &yb = y[t][NACC - 1];
                dmma(ya.x, ya.y, q[t][i].x, vb.x);
                dmma(yb.x, yb.y, q[t][i].y, vb.y);
            }
        }
        double2 w[NCT];
#pragma unroll
        for (int t = 0; t < NCT; t++) {
            w[t] = y[t][0];
            if (NACC == 2) {
                w[t].x += y[t][1].x;
                w[t].y += y[t][1].y;
            }
        }
        // Q_W^T += W^T V_g^T
#pragma unroll
        for (int i = 0; i < LAM; i++) {
            const double2 ub = updB[i * 32 + lane];
#pragma unroll
            for (int t = 0; t < NCT; t++) {
                dmma(q[t][i].x, q[t][i].y, w[t].x, ub.x);
                dmma(q[t][i].x, q[t][i].y, w[t].y, ub.y);
            }
        }
    }
};

// Complex Hermitian case (NEXT-3, R15) on FP64 tensor cores.  The window holds
// NCT/2 complex 8-column tiles as real tile pairs q[2u] = Re, q[2u+1] = Im.  The group applies
// M = H_7 ... H_0 (H_a = I - tau_a v_a v_a^H, a = 0 first) = I - V T'^H V^H, T' the forward
// compact-WY factor of conj(tau); with U' = -V T' (prep):  W = U'^H Q_W,  Q_W += V W, i.e.
//   W^T = Q^T conj(U'):  Re = Qr^T Ur + Qi^T Ui,   Im = Qi^T Ur - Qr^T Ui
//   Q^T += W^T V^T:      Qr += Wr Vr - Wi Vi,      Qi += Wr Vi + Wi Vr
// 8*LAM + 8*LAM DMMA.8x8x4 per complex tile (4x the real count for 4x the flops).  Blob
// (prep_zmma_kernel): B-fragments of Re U', Im U', Re V, Im V, each [LAM][32 lanes][2].
template <int LAM, int NCT>
struct ZmmaGroup {
    static constexpr int BLOB = 256 * LAM;
    static constexpr int NZ = NCT / 2;
    __device__ __forceinline__ static void apply(double2 (&q)[NCT][LAM], const double *blob, uint32_t,
                                                 int lane) {
        const double2 *dUr = reinterpret_cast<const double2 *>(blob);
        const double2 *dUi = dUr + 32 * LAM;
        const double2 *uVr = dUr + 64 * LAM;
        const double2 *uVi = dUr + 96 * LAM;
        double2 ya[NZ], yb[NZ], yc[NZ], yd[NZ];            // Qr.Ur, Qi.Ui, Qi.Ur, Qr.Ui
#pragma unroll
        for (int u = 0; u < NZ; u++) ya[u] = yb[u] = yc[u] = yd[u] = make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < LAM; i++) {
            const double2 ur = dUr[i * 32 + lane], ui = dUi[i * 32 + lane];
#pragma unroll
            for (int u = 0; u < NZ; u++) {
                const double2 qr = q[2 * u][i], qi = q[2 * u + 1][i];
                dmma(ya[u].x, ya[u].y, qr.x, ur.x);
                dmma(yb[u].x, yb[u].y, qi.x, ui.x);
                dmma(yc[u].x, yc[u].y, qi.x, ur.x);
                dmma(yd[u].x, yd[u].y, qr.x, ui.x);
                dmma(ya[u].x, ya[u].y, qr.y, ur.y);
                dmma(yb[u].x, yb[u].y, qi.y, ui.y);
                dmma(yc[u].x, yc[u].y, qi.y, ur.y);
                dmma(yd[u].x, yd[u].y, qr.y, ui.y);
            }
        }
        double2 wr[NZ], wi[NZ], nwi[NZ];
#pragma unroll
        for (int u = 0; u < NZ; u++) {
            wr[u] = make_double2(ya[u].x + yb[u].x, ya[u].y + yb[u].y);
            wi[u] = make_double2(yc[u].x - yd[u].x, yc[u].y - yd[u].y);
            nwi[u] = make_double2(-wi[u].x, -wi[u].y);
        }
#pragma unroll
        for (int i = 0; i < LAM; i++) {
            const double2 vr = uVr[i * 32 + lane], vi = uVi[i * 32 + lane];
#pragma unroll
            for (int u = 0; u < NZ; u++) {
                double2 &qr = q[2 * u][i];
                double2 &qi = q[2 * u + 1][i];
                dmma(qr.x, qr.y, wr[u].x, vr.x);
                dmma(qi.x, qi.y, wr[u].x, vi.x);
                dmma(qr.x, qr.y, wr[u].y, vr.y);
                dmma(qi.x, qi.y, wr[u].y, vi.y);
                dmma(qr.x, qr.y, nwi[u].x, vi.x);
                dmma(qi.x, qi.y, wi[u].x, vr.x);
                dmma(qr.x, qr.y, nwi[u].y, vi.y);
                dmma(qi.x, qi.y, wi[u].y, vr.y);
            }
        }
    }
};

template <int KIND, int LAM, int NCT>
using GroupOf = typename std::conditional<KIND == KIND_DMMA, DmmaGroup<LAM, NCT>, ZmmaGroup<LAM, NCT>>::type;

// Complex Q I/O (interleaved re/im doubles): a lane's complex rows r, r+1 of one column as the
// real tile pair (Re rows r, r+1), (Im rows r, r+1); rows outside [0, n) read as zero and are
// never written.  The async form lands the raw rows (re_r, im_r), (re_r+1, im_r+1) in two
// 16-byte slots; zsplit turns them into the pair.
__device__ __forceinline__ void zload_pair(const double *colp, bool ok, int n, int r, double2 &re, double2 &im) {
    double2 a = make_double2(0.0, 0.0), b = make_double2(0.0, 0.0);
    if (ok && r >= 0 && r < n) {
        a = *reinterpret_cast<const double2 *>(colp + 2 * r);
        if (r + 1 < n) b = *reinterpret_cast<const double2 *>(colp + 2 * r + 2);
    }
    re = make_double2(a.x, b.x);
    im = make_double2(a.y, b.y);
}
__device__ __forceinline__ void zload_pair_async(double2 *da, double2 *db, const double *colp, bool ok, int n, int r) {
    const bool ia = ok && r >= 0 && r < n, ib = ok && r >= 0 && r + 1 < n;
    cp_async16_zfill(da, ia ? colp + 2 * r : colp, ia ? 16u : 0u);
    cp_async16_zfill(db, ib ? colp + 2 * r + 2 : colp, ib ? 16u : 0u);
}
__device__ __forceinline__ void zsplit(double2 a, double2 b, double2 &re, double2 &im) {
    re = make_double2(a.x, b.x);
    im = make_double2(a.y, b.y);
}
__device__ __forceinline__ void zstore_pair(double *colp, bool ok, int n, int r, double2 re, double2 im) {
    if (ok && r >= 0 && r < n) {
        *reinterpret_cast<double2 *>(colp + 2 * r) = make_double2(re.x, im.x);
        if (r + 1 < n) *reinterpret_cast<double2 *>(colp + 2 * r + 2) = make_double2(re.y, im.y);
    }
}

template <int KIND, int B8, int D, int CW, int NCT, int K>
struct DmmaCfg {
    static constexpr int LAM = B8 + 1;
    using Group = GroupOf<KIND, LAM, NCT>;
    static constexpr int BLOB = Group::BLOB;               // doubles per prepared group
    static constexpr int NWARP = D * CW;
    static constexpr int THREADS = 32 * NWARP;
    static constexpr int ZF = (KIND == KIND_ZMMA) ? 2 : 1;  // real tiles per (complex) tile
    static constexpr int T = CW * NCT / ZF;                // 8-column tiles per work item
    static constexpr int STAGES = (K * D * BLOB * 8 * 3 <= 100 * 1024) ? 3 : 2;
    // shared memory: STAGES x K x D fragment blobs, hand-off chunks [2][D][K][CW][NCT][32],
    // warp-0 intake chunks [2][K][CW][NCT][32], barriers + the dequeued item index
    static constexpr size_t SMEM_BLOBS = size_t(STAGES) * K * D * BLOB * sizeof(double);
    static constexpr size_t SMEM_HAND = size_t(2) * D * K * CW * NCT * 64 * sizeof(double);
    static constexpr size_t SMEM_INTAKE = size_t(2) * K * CW * NCT * 64 * sizeof(double);
    static constexpr size_t SMEM = SMEM_BLOBS + SMEM_HAND + SMEM_INTAKE + 64;
    // Occupancy intent as a launch bound: the register window (4*LAM*NCT) + ~80, so an
    // incidental code change cannot let ptxas spread into a CTA/SM fewer (seen: 138 -> 183
    // registers, 3 -> 2 CTAs/SM, 28.1 -> 21.0 TF/s).
    static constexpr int REG_EST = 4 * LAM * NCT + 80 + (KIND == KIND_ZMMA ? 16 : 0);
    static constexpr int MINB_RAW = 65536 / (THREADS * REG_EST);
    static constexpr int MINB = MINB_RAW < 1 ? 1 : (MINB_RAW > 8 ? 8 : MINB_RAW);
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
//
// Inside an item, group-time tau = 0, 1, ...: depth warp d applies group
// g = G - 1 - tau + d*(K+1) of depth m0 + d; its window's top chunk is C0 - tau + d*(LAM + K).
// Depth m0+d+1 trails depth m0+d by K+1 groups, so the chunk warp d takes in after tau was
// emitted by warp d-1 after tau - K, i.e. in the previous step: the K chunks between two
// windows are in transit in shared memory.  One step = K group-times = one CTA barrier.
template <int KIND, int B8, int D, int CW, int NCT, int K>
__global__ void __launch_bounds__(DmmaCfg<KIND, B8, D, CW, NCT, K>::THREADS, DmmaCfg<KIND, B8, D, CW, NCT, K>::MINB)
apply_dmma_kernel(int64_t n64, int64_t nev64, const double *__restrict__ blobs, double *Q, int64_t ldq,
                  uint64_t *prog, int pub_period) {
    using Cfg = DmmaCfg<KIND, B8, D, CW, NCT, K>;
    constexpr int LAM = Cfg::LAM;
    constexpr int BLOB = Cfg::BLOB;
    constexpr int S = Cfg::STAGES;
    constexpr int T = Cfg::T;
    constexpr int ZF = Cfg::ZF;
    constexpr int B = 8 * B8;
    constexpr int LAG = K + 1;                             // groups depth m+1 trails depth m
    constexpr int SPAN = LAM + K;                          // chunk distance between stacked windows

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *sblob = reinterpret_cast<double *>(smem_raw);                                        // [S][K][D][BLOB]
    double2 *shand = reinterpret_cast<double2 *>(smem_raw + Cfg::SMEM_BLOBS);                    // [2][D][K][CW][NCT][32]
    double2 *sintake = reinterpret_cast<double2 *>(smem_raw + Cfg::SMEM_BLOBS + Cfg::SMEM_HAND);  // [2][K][CW][NCT][32]
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + Cfg::SMEM_BLOBS + Cfg::SMEM_HAND + Cfg::SMEM_INTAKE);
    uint64_t *ebars = bars + S;                            // per-stage "consumed" barriers (ring mode)
    int *s_item = reinterpret_cast<int *>(bars + 2 * S);
    // Ring mode (one depth warp row, one group per step, 3+ stages): no CTA barrier per step.
    // Every warp arrives on the stage's "consumed" mbarrier after its group; the issuer refills a
    // stage only after all warps consumed its previous use, one step of slack behind (fragments
    // are issued AHEAD = S-2 steps ahead).  CTA barriers remain on publish steps (progress words)
    // and at item boundaries.
    constexpr bool kRing = (D == 1 && K == 1 && S >= 3);
    constexpr int AHEAD = kRing ? S - 2 : S - 1;

    const int n = int(n64), nev = int(nev64);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int d = warp / CW, cw = warp % CW;
    const int M = int(num_depths(n64, B));
    const int C0 = (n - 2) >> 3;                           // top chunk of every depth's first window
    const int ntile = (nev + 7) >> 3;
    const int NX = (ntile + T - 1) / T;
    const int NP = (M + D - 1) / D;
    const int rsub = 2 * (lane & 3);
    constexpr uint32_t kAllTiles = (1u << NCT) - 1u;
    // hand-off / intake slot of (parity, j, t) for this lane
    auto hslot = [&](int par, int dd, int j, int t) {
        return ((((par * D + dd) * K + j) * CW + cw) * NCT + t) * 32 + lane;
    };
    auto islot = [&](int par, int j, int t) { return (((par * K + j) * CW + cw) * NCT + t) * 32 + lane; };
    // the fragment ring is fed by the last warp (deepest depth row: no HBM intake when D > 1;
    // with D = 1 it spares warp 0, which also dequeues items and publishes progress)
    const bool issuer = threadIdx.x == 32 * (D * CW - 1);

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; i++) mbar_init(&bars[i], 1);
        for (int i = 0; i < S; i++) mbar_init(&ebars[i], D * CW);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    uint32_t phase_bits = 0;  // parity of the next completion, per stage (all threads track it)
    int stage0 = 0;           // ring stage of the item's step 0
    int gstep0 = 0;           // global step index of the item's step 0 (ring mode)

    for (;;) {
        if (threadIdx.x == 0)
            *s_item = int(atomicAdd(reinterpret_cast<unsigned long long *>(prog + int64_t(NX) * NP), 1ull));
        __syncthreads();
        const int k = *s_item;
        if (k >= NX * NP) break;
        const int p = k / NX, x = k % NX;
        const int m0 = p * D;
        const int tile_end = min(ntile, (x + 1) * T);
        double *qcol[NCT];
        uint32_t okmask = 0, tilemask = 0;
#pragma unroll
        for (int t = 0; t < NCT; t++) {
            const int tile = x * T + cw * (NCT / ZF) + t / ZF;
            const int c = tile * 8 + (lane >> 2);
            if (tile < tile_end) tilemask |= 1u << t;
            if (tile < tile_end && c < nev) okmask |= 1u << t;
            qcol[t] = Q + int64_t(ZF) * int64_t(min(c, nev - 1)) * ldq;
        }
        const int G = int(groups_at_depth(n64, B8, m0));
        const int dmax = min(D, M - m0) - 1;
        const int NT = G + dmax * LAG;                     // group-times of this item
        const int nsteps = (NT + K - 1) / K;

        // publish steps: every pub_period steps (host-chosen) and the step whose emission
        // finalises chunk C0 (a next pass waiting for its first window starts at once); only
        // while the deepest warps' emissions are real chunks
        int pub_count = 0;                                 // == st % pub_period
        auto pub_step = [&](int st) {
            const int cbot = C0 - (st * K + K - 1) + (D - 1) * SPAN + LAM - 1;
            return (pub_count == pub_period - 1 || cbot == C0) && cbot <= C0 + 1 && cbot >= 0;
        };
        auto group_valid = [&](int tau, int dd) {
            const int g = G - 1 - tau + dd * LAG;
            return dd <= dmax && tau < NT && g >= 0 && g < G - dd * B8;
        };
        // blob of group g at depth m0 + dd: bbase[dd] + g * BLOB (64-bit bases, once per item)
        const double *bbase[D];
#pragma unroll
        for (int dd = 0; dd < D; dd++) bbase[dd] = blobs + group_base(n64, B8, m0 + dd) * BLOB;
        auto issue = [&](int st) {  // fragments of step st -> ring stage (stage0 + st) % S
            const int stg = (stage0 + st) % S;
            uint64_t *bar = &bars[stg];
            if constexpr (kRing) {                          // previous use of this stage consumed?
                const int g = gstep0 + st;
                if (g >= S) mbar_wait(&ebars[stg], uint32_t(((g / S) - 1) & 1));
            }
            uint32_t bytes = 0;
            for (int j = 0; j < K; j++)
                for (int dd = 0; dd <= dmax; dd++)
                    if (group_valid(st * K + j, dd)) bytes += BLOB * 8;
            mbar_arrive_expect_tx(bar, bytes);
            for (int j = 0; j < K; j++)
                for (int dd = 0; dd <= dmax; dd++)
                    if (group_valid(st * K + j, dd)) {
                        const int g = G - 1 - (st * K + j) + dd * LAG;
                        bulk_g2s(sblob + ((stg * K + j) * D + dd) * BLOB, bbase[dd] + int64_t(g) * BLOB, BLOB * 8, bar);
                    }
        };
        if (issuer)
            for (int st = 0; st < AHEAD && st < nsteps; st++) issue(st);

        // cross-pass dependency (warp 0 only): chunk c must be final from pass p-1
        uint32_t seen = 0;
        auto await_chunk = [&](int c) {
            if (p == 0 || c < 0) return;
            const uint32_t need = uint32_t(C0 + 2 - c);
            if (seen >= need) return;
            if (lane == 0) {
                uint64_t v = ld_acquire_u64(prog + (k - NX));
                ELPA_WATCHDOG_START();
                while (v < need) {
                    __nanosleep(128);
                    v = ld_acquire_u64(prog + (k - NX));
                    ELPA_WATCHDOG_CHECK();
                }
                seen = v > 0xFFFFFFFFull ? 0xFFFFFFFFu : uint32_t(v);
            }
            seen = __shfl_sync(0xffffffffu, seen, 0);
        };
        // warp 0 streams its new top chunks HBM -> shared (cp.async, one step ahead): the chunk
        // entering after group-time tau = st*K + j is C0 - tau - 1, in slot [st & 1][j]
        auto intake = [&](int st) {
#pragma unroll
            for (int j = 0; j < K; j++) {
                const int c = C0 - (st * K + j) - 1;
                await_chunk(c);
                if (ZF == 1 && okmask == kAllTiles && c >= 0 && 8 * c + 8 <= n) {
                    // interior chunk, every column valid: no bounds logic
#pragma unroll
                    for (int t = 0; t < NCT; t++)
                        cp_async16_zfill(&sintake[islot(st & 1, j, t)], qcol[t] + 8 * c + rsub, 16u);
                } else {
#pragma unroll
                    for (int t = 0; t < NCT; t += ZF) {
                        if constexpr (ZF == 2)
                            zload_pair_async(&sintake[islot(st & 1, j, t)], &sintake[islot(st & 1, j, t + 1)],
                                             qcol[t], (okmask >> t) & 1, n, 8 * c + rsub);
                        else
                            load_pair_async(&sintake[islot(st & 1, j, t)], qcol[t], (okmask >> t) & 1, n,
                                            8 * c + rsub);
                    }
                }
            }
            cp_async_commit();
        };

        // chunk I/O of all NCT tiles (complex: tile pairs, interleaved storage)
        auto load_chunk = [&](double2 (&qq)[NCT][LAM], int i, int r) {
#pragma unroll
            for (int t = 0; t < NCT; t += ZF) {
                if constexpr (ZF == 2) zload_pair(qcol[t], (okmask >> t) & 1, n, r, qq[t][i], qq[t + 1][i]);
                else qq[t][i] = load_pair(qcol[t], (okmask >> t) & 1, n, r);
            }
        };
        auto store_tiles = [&](const double2 *v, int r) {      // v[t], t < NCT
            if (ZF == 1 && okmask == kAllTiles && r >= 0 && r + 2 <= n) {   // no bounds logic
#pragma unroll
                for (int t = 0; t < NCT; t++) *reinterpret_cast<double2 *>(qcol[t] + r) = v[t];
                return;
            }
#pragma unroll
            for (int t = 0; t < NCT; t += ZF) {
                if constexpr (ZF == 2) zstore_pair(qcol[t], (okmask >> t) & 1, n, r, v[t], v[t + 1]);
                else store_pair(qcol[t], (okmask >> t) & 1, n, r, v[t]);
            }
        };
        double2 q[NCT][LAM];
        if (d == 0) await_chunk(C0);
#pragma unroll
        for (int i = 0; i < LAM; i++) load_chunk(q, i, 8 * (C0 + d * SPAN + i) + rsub);
        if (d == 0) intake(0);

        bool done = false;
        for (int st = 0; !done; st++) {
            if (issuer && st + AHEAD < nsteps) issue(st + AHEAD);
            if (d == 0 && st + 1 < nsteps) intake(st + 1);
            const uint32_t stage = uint32_t((stage0 + st) % S);
            const uint32_t par = (phase_bits >> stage) & 1u;
            phase_bits ^= (1u << stage);
            bool waited = false;
#pragma unroll 1
            for (int j = 0; j < K; j++) {
                const int tau = st * K + j;
                if (group_valid(tau, d)) {
                    if (!waited) { mbar_wait(&bars[stage], par); waited = true; }
                    Cfg::Group::apply(q, sblob + ((stage * K + j) * D + d) * BLOB, tilemask, lane);
                }
                if constexpr (kRing) {                      // this warp is done with the stage
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&ebars[stage]);
                }
                if (tau + 1 >= NT) { done = true; break; }     // final windows written back below
                // emit the bottom chunk: to HBM (deepest warp) or to warp d+1 for the next step
                const int cbot = C0 - tau + d * SPAN + LAM - 1;
                if (d == D - 1) {
                    double2 bot[NCT];
#pragma unroll
                    for (int t = 0; t < NCT; t++) bot[t] = q[t][LAM - 1];
                    store_tiles(bot, 8 * cbot + rsub);
                    // on publish steps the emitted stores are fenced here; thread 0 publishes after
                    // the step barrier, when EVERY column warp of the item has stored its chunks.
                    // (Dropping this fence and relying on bar.sync + thread 0's release alone
                    // measured 1.5x slower for D = 1 shapes: 28 -> 18.5 TF/s at C3.)
                    if (pub_step(st)) __threadfence();
                } else {
#pragma unroll
                    for (int t = 0; t < NCT; t++) shand[hslot(st & 1, d + 1, j, t)] = q[t][LAM - 1];
                }
                // shift the window one chunk; the new top chunk arrived during the previous step
                if (d == 0 && j == 0) cp_async_wait<1>();
#pragma unroll
                for (int t = 0; t < NCT; t++) {
#pragma unroll
                    for (int i = LAM - 1; i > 0; i--) q[t][i] = q[t][i - 1];
                    if constexpr (ZF == 2) {
                        // complex: tile t+1 is shifted in the next iteration, so the (Re, Im) pair
                        // is split when its odd member is reached
                        if (d == 0 && (t & 1)) {
                            zsplit(sintake[islot(st & 1, j, t - 1)], sintake[islot(st & 1, j, t)], q[t - 1][0],
                                   q[t][0]);
                            continue;
                        }
                        if (d == 0) continue;
                    }
                    if (d == 0) {
                        q[t][0] = sintake[islot(st & 1, j, t)];
                    } else if (st > 0) {
                        q[t][0] = shand[hslot((st + 1) & 1, d, j, t)];
                    } else {
                        q[t][0] = make_double2(0.0, 0.0);   // rows below the matrix (chunk >= C0 + 2)
                    }
                }
            }
            if (done) break;
            if (!kRing || pub_step(st)) __syncthreads();
            if (threadIdx.x == 0 && pub_step(st)) {
                // every chunk >= the deepest warps' last emission is final for the next pass
                const int cbot = C0 - (st * K + K - 1) + (D - 1) * SPAN + LAM - 1;
                st_release_u64(prog + k, uint64_t(C0 + 2 - cbot));
            }
            pub_count = (pub_count == pub_period - 1) ? 0 : pub_count + 1;
        }
        if (d == 0) cp_async_wait<0>();   // drain any unused intake before slot reuse
        __syncthreads();                  // the last step's hand-off writes are visible below
        // write back the final windows: top chunk C0 - (NT - 1) + d*SPAN
#pragma unroll
        for (int i = 0; i < LAM; i++) {
            double2 col[NCT];
#pragma unroll
            for (int t = 0; t < NCT; t++) col[t] = q[t][i];
            store_tiles(col, 8 * (C0 - (NT - 1) + d * SPAN + i) + rsub);
        }
        // chunks in transit between windows (emitted by warp d-1, not yet taken by warp d) are final
        if (d >= 1) {
            const int st = (NT - 1) / K;                   // step of the last group-time
            const int jl = (NT - 1) % K;
            for (int j = jl; j < K && st > 0; j++) {      // emitted in the previous step
                const int c = C0 - ((st - 1) * K + j) + (d - 1) * SPAN + LAM - 1;
                double2 h[NCT];
#pragma unroll
                for (int t = 0; t < NCT; t++) h[t] = shand[hslot((st + 1) & 1, d, j, t)];
                store_tiles(h, 8 * c + rsub);
            }
            for (int j = 0; j < jl; j++) {                // emitted in this step before the last group-time
                const int c = C0 - (st * K + j) + (d - 1) * SPAN + LAM - 1;
                double2 h[NCT];
#pragma unroll
                for (int t = 0; t < NCT; t++) h[t] = shand[hslot(st & 1, d, j, t)];
                store_tiles(h, 8 * c + rsub);
            }
        }
        __threadfence();
        __syncthreads();  // item complete: publish, and the smem ring/hand-off are free again
        if (threadIdx.x == 0) st_release_u64(prog + k, kPassDone);
        stage0 = (stage0 + nsteps) % S;
        gstep0 += nsteps;
    }
}

}  // namespace elpa_b200
