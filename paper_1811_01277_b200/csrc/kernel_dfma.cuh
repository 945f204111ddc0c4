// kernel_dfma.cuh — the FP64 CUDA-core (DFMA) formulation of the hot path that BASELINE.json's
// north_star item (3) describes, built as the measured alternative to the tensor-core (DMMA)
// kernel: "each CTA owns a coalesced column stripe of Q and streams the sweep's row window ...
// reflectors are fused in groups of k = 2/4/6/8 so each Q tile is reused k times ... reflectors
// double-buffered into shared memory".  The ELPA kernels the paper speeds up apply 2/4/6
// reflectors per pass in AVX-512 registers (prior art); here:
//   * two lanes own one column of Q (16 columns per warp, CW warps per CTA), each holding half
//     of the column's window rows in registers (row pairs, alternating between the two lanes):
//     one lane cannot hold the nbw + k FP64 rows of its window without spilling at nbw = 64;
//   * group g of depth m holds the KF sweeps j = KF*g + KF-2-a, a = 0..KF-1 (a = 0 is the
//     highest sweep, applied first: reverse generation order within the group).  Reflector a
//     starts at row KF*g + m*b + KF-1-a, so the group's rows are the window
//     [KF*g + m*b, KF*g + m*b + WP), WP >= b + KF;
//   * the KF reflectors are applied one at a time, exactly the oracle's recurrence per column
//     (w = tau v^T q, q -= w v) but with fused multiply-adds: each lane forms its half of v^T q,
//     one shuffle adds the halves, and each lane updates its rows.  Every window row is loaded
//     from HBM once per group and reused by the KF reflectors — the k-fold reuse of the paper's
//     blocked kernels — with no compact-WY factor;
//   * v is laid out in the blob aligned to the window (zero outside the reflector) and read with
//     warp-broadcast 16-byte shared-memory loads (two rows per load, re-read for the update);
//   * groups run from the bottom of the matrix upward (g descending), the window sliding up by
//     KF rows per group; the window is a register ring (no moves): the KF new top rows are
//     prefetched one step ahead, the KF bottom rows are written back.
// Work items, the dynamic dequeue and the progress words are those of the DMMA kernel
// with one depth per item: item (x, m) consumes the rows item (x, m-1) has
// finalised.  Progress is counted in rows: prog = n - r means every row >= r is final.
#pragma once
#include "kernel_dmma.cuh"

namespace elpa_b200 {

// window rows: the smallest multiple of k that is >= b + k and a multiple of 4 (the row-pair
// ring is split evenly between the two lanes of a column)
__host__ __device__ constexpr int dfma_window(int b, int kf) {
    int w = (b + kf + kf - 1) / kf * kf;
    while (w % 4) w += kf;
    return w;
}
// doubles per prepared group: per reflector the window-aligned vector twice over (2 WP: the
// lanes' pair sequences wrap around the ring without an index wrap), then tau[KF], padded even
__host__ __device__ constexpr int dfma_blob_doubles(int b, int kf) {
    return kf * 2 * dfma_window(b, kf) + kf + (kf & 1);
}

// groups of depth m (sweeps j <= J_m = n-3-m*b, group g covers j <= KF*g + KF-2)
__host__ __device__ inline int64_t dfma_groups(int64_t n, int64_t b, int64_t kf, int64_t m) {
    const int64_t x = n - 1 - m * b;                       // = J_m + 2
    return x > 0 ? (x + kf - 1) / kf : 0;
}

// gbase[m] = sum_{m' < m} groups(m'), m = 0..M (one thread: M is at most a few thousand)
__global__ void dfma_gbase_kernel(int64_t n, int64_t b, int64_t kf, int64_t M, int64_t *gbase) {
    int64_t acc = 0;
    for (int64_t m = 0; m <= M; m++) {
        gbase[m] = acc;
        if (m < M) acc += dfma_groups(n, b, kf, m);
    }
}

// one thread per blob element of the groups [g_lo, g_hi); grid (element blocks, M).  Reflector a's vector occupies window
// rows [KF-1-a, KF-1-a+L) (v_0 = 1), zero elsewhere, stored at [a*2WP, a*2WP + WP) and again at
// [a*2WP + WP, (a+1)*2WP).
template <int B, int KF>
__global__ void __launch_bounds__(256)
prep_dfma_kernel(int64_t n, const double *__restrict__ hh_v, const double *__restrict__ hh_tau,
                 const int64_t *__restrict__ gbase, double *__restrict__ blobs, int64_t g_lo, int64_t g_hi) {
    constexpr int WP = dfma_window(B, KF);
    constexpr int BLOB = dfma_blob_doubles(B, KF);
    const int64_t m = blockIdx.y;
    const int64_t G = dfma_groups(n, B, KF, m);
    const int64_t Jm = n - 3 - m * B;
    double *base = blobs + gbase[m] * BLOB;
    const int64_t e1 = (g_hi < G ? g_hi : G) * BLOB;      // groups [g_lo, g_hi) of this depth
    for (int64_t e = g_lo * BLOB + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < e1;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t g = e / BLOB;
        const int w = int(e % BLOB);
        double val = 0.0;
        if (w < KF * 2 * WP) {
            const int a = w / (2 * WP), row = (w % (2 * WP)) % WP;
            const int i = row - (KF - 1 - a);               // index into the reflector's vector
            const int64_t j = KF * g + KF - 2 - a;
            if (j >= 0 && j <= Jm && i >= 0) {
                const int64_t s = j + 1 + m * B;
                const int64_t L = (n - s < B) ? (n - s) : B;
                if (i < L) val = (i == 0) ? 1.0 : hh_v[(hh_off(j, n, B) + m) * B + i];
            }
        } else if (w < KF * 2 * WP + KF) {
            const int a = w - KF * 2 * WP;
            const int64_t j = KF * g + KF - 2 - a;
            if (j >= 0 && j <= Jm) val = hh_tau[hh_off(j, n, B) + m];
        }
        base[e] = val;
    }
}

// 16-byte shared-memory load that the compiler may neither merge with an earlier load of the
// same address nor hoist ahead of the previous one: the update pass re-reads v instead of
// keeping the b values of the dot pass live (b more registers: spills at b = 64)
__device__ __forceinline__ double2 lds_v2(const double2 *p) {
    double2 v;
    asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
    return v;
}

// compile-time loop: f(integral_constant<int, I>) for I = I0 .. I1-1
template <int I0, int I1, class F>
__device__ __forceinline__ void dfma_static_for(F &&f) {
    if constexpr (I0 < I1) {
        f(std::integral_constant<int, I0>{});
        dfma_static_for<I0 + 1, I1>(f);
    }
}

template <int B, int KF, int CW>
struct DfmaCfg {
    static constexpr int WP = dfma_window(B, KF);           // window rows
    static constexpr int NPR = WP / 2;                      // row pairs of the window (ring slots)
    static constexpr int NL = NPR / 2;                      // ring slots per lane
    static constexpr int NW = WP / KF;                      // steps a row spends in the window
    static constexpr int BLOB = dfma_blob_doubles(B, KF);
    static constexpr int THREADS = 32 * CW;
    static constexpr int COLS = 16 * CW;                    // columns per CTA (two lanes per column)
    static constexpr int STAGES = 4;                        // blobs issued 2 steps ahead, 1 step slack
    static constexpr size_t SMEM = size_t(STAGES) * BLOB * sizeof(double) + 2 * STAGES * 8 + 16;   // + barriers, item
};

template <int B, int KF, int CW>
__global__ void __launch_bounds__((DfmaCfg<B, KF, CW>::THREADS))
apply_dfma_kernel(int64_t n64, int64_t nev64, const double *__restrict__ blobs, const int64_t *__restrict__ gbase,
                  double *Q, int64_t ldq, uint64_t *prog, int pub_period) {
    using Cfg = DfmaCfg<B, KF, CW>;
    constexpr int WP = Cfg::WP, NPR = Cfg::NPR, NL = Cfg::NL, NW = Cfg::NW;
    constexpr int BLOB = Cfg::BLOB;
    constexpr int S = Cfg::STAGES;
    constexpr int KP = KF / 2;                              // row pairs per step

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *sblob = reinterpret_cast<double *>(smem_raw);                                  // [S][BLOB]
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + size_t(S) * BLOB * sizeof(double));
    uint64_t *ebars = bars + S;
    int *s_item = reinterpret_cast<int *>(ebars + S);

    const int n = int(n64), nev = int(nev64);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int h = lane & 1;                                 // which half of the column's rows
    const int M = int(num_depths(n64, B));
    const int NX = (nev + Cfg::COLS - 1) / Cfg::COLS;
    const bool issuer = threadIdx.x == 32 * (CW - 1);

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; i++) mbar_init(&bars[i], 1);
        for (int i = 0; i < S; i++) mbar_init(&ebars[i], CW);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    int gstep0 = 0;                                         // ring position of the item's step 0

    for (;;) {
        if (threadIdx.x == 0)
            *s_item = int(atomicAdd(reinterpret_cast<unsigned long long *>(prog + int64_t(NX) * M), 1ull));
        __syncthreads();
        const int k = *s_item;
        if (k >= NX * M) break;
        const int m = k / NX, x = k % NX;
        const int c = x * Cfg::COLS + warp * 16 + (lane >> 1);
        const bool ok = c < nev;
        double *qc = Q + int64_t(ok ? c : nev - 1) * ldq;
        const int G = int(dfma_groups(n64, B, KF, m));
        const int rowbase = m * B;                          // window top of group g: KF*g + rowbase
        const double *bbase = blobs + gbase[m] * BLOB;

        auto issue = [&](int st) {                          // blob of step st (group G-1-st)
            const int gs = gstep0 + st, stg = gs % S;
            if (gs >= S) mbar_wait(&ebars[stg], uint32_t(((gs / S) - 1) & 1));
            mbar_arrive_expect_tx(&bars[stg], BLOB * 8);
            bulk_g2s(sblob + stg * BLOB, bbase + int64_t(G - 1 - st) * BLOB, BLOB * 8, &bars[stg]);
        };
        constexpr int AHEAD = S - 2;
        if (issuer)
            for (int st = 0; st < AHEAD && st < G; st++) issue(st);

        uint64_t seen = 0;
        auto await_rows = [&](int r) {                      // every row >= r final from depth m-1
            if (m == 0 || r >= n) return;                   // rows past the matrix need no producer
            const uint64_t need = uint64_t(n - max(r, 0));
            if (seen >= need) return;
            if (lane == 0) {
                uint64_t v = ld_acquire_u64(prog + (k - NX));
                ELPA_WATCHDOG_START();
                while (v < need) {
                    __nanosleep(256);
                    v = ld_acquire_u64(prog + (k - NX));
                    ELPA_WATCHDOG_CHECK();
                }
                seen = v;
            }
            seen = __shfl_sync(0xffffffffu, seen, 0);
        };
        auto ld = [&](int r) { return (ok && r >= 0 && r < n) ? qc[r] : 0.0; };
        // row pair (r, r+1): one 16-byte access when inside the matrix and aligned (ldq even, r
        // even: always true of the window rows when nbw and k are even), else per element
        auto ld_pair = [&](int r) {
            if (ok && r >= 0 && r + 2 <= n && ((reinterpret_cast<uintptr_t>(qc + r) & 15) == 0))
                return *reinterpret_cast<const double2 *>(qc + r);
            return make_double2(ld(r), ld(r + 1));
        };
        auto st_pair = [&](int r, double2 v) {
            if (!ok) return;
            if (r >= 0 && r + 2 <= n && ((reinterpret_cast<uintptr_t>(qc + r) & 15) == 0)) {
                *reinterpret_cast<double2 *>(qc + r) = v;
            } else {
                if (r >= 0 && r < n) qc[r] = v.x;
                if (r + 1 >= 0 && r + 1 < n) qc[r + 1] = v.y;
            }
        };
        // publish early once the emitted rows cover the next depth's first window (its item can
        // start), then every pub_period steps
        const int next_top0 = (m + 1 < M) ? KF * int(dfma_groups(n64, B, KF, m + 1) - 1) + (m + 1) * B : -1;
        bool early = m + 1 < M;

        // Time steps t = 0 .. G + 2*NW - 2 (uniform per-step code: every Q row enters and leaves
        // the window through the KF-row intake and emission, no bulk window load/store):
        //   window top(t) = rowbase + KF*(G - 1 + NW - t); group g = G - 1 - (t - NW) is applied
        //   at step t when 0 <= g < G;
        //   t < NW: warm-up (the window starts wholly past row n - 1, all zero, and fills from
        //   below: by step NW every chunk came through the intake);
        //   after the group-0 step, NW - 1 drain steps emit the last window (zeros enter the top:
        //   rows above rowbase belong to earlier depths and are never read or written here).
        // Ring: window row pair p of step t lives in slot s = (p - KP*t) mod NPR, slot s in lane
        // (s & 1) of the column's lane pair at qh[s >> 1].  Lane h's slots 2l + h hold window pairs
        // p = (2l + h + KP*r) mod NPR (r = t mod NW), i.e. v pairs c0 + 2l with c0 = (h + KP*r)
        // mod NPR, read from the doubled vector without an index wrap.  The step loop is unrolled
        // NW times so every ring index is a compile-time constant.
        double2 qh[NL];
#pragma unroll
        for (int i = 0; i < NL; i++) qh[i] = make_double2(0.0, 0.0);
        const int T = G + 2 * NW - 1;                       // steps of this item
        int top = rowbase + KF * (G - 1 + NW);
        double2 nxt[KP];                                    // the next step's top pairs (own slots only)
        auto fetch = [&](auto rc_next, int t) {             // intake for step t (t >= 1), rotation of t
            constexpr int r = decltype(rc_next)::value;
            const int rr = top - KF;                        // top(t) = top(t-1) - KF
            const bool real = t <= G - 1 + NW;              // the group-0 step takes in real rows
            if (real) await_rows(rr);
#pragma unroll
            for (int i = 0; i < KP; i++) {
                const int s = ((i - KP * r) % NPR + NPR) % NPR;
                nxt[i] = (real && (s & 1) == h) ? ld_pair(rr + 2 * i) : make_double2(0.0, 0.0);
            }
        };
        if (T > 1) fetch(std::integral_constant<int, 1 % NW>{}, 1);
        int pub_count = 0;
        auto step = [&](auto rc, int t) {
            constexpr int r = decltype(rc)::value;          // ring rotation of step t (t mod NW)
            auto slot = [](int p) { return ((p - KP * r) % NPR + NPR) % NPR; };
            if (t > 0) {                                    // slide up by KF rows: take in the top pairs
#pragma unroll
                for (int i = 0; i < KP; i++) {
                    const int s = slot(i);
                    if ((s & 1) == h) qh[s >> 1] = nxt[i];
                }
                top -= KF;
                if (t + 1 < T) fetch(std::integral_constant<int, (r + 1) % NW>{}, t + 1);
            }
            const int g = G - 1 - (t - NW);
            if (g >= 0 && g < G) {
                const int st = G - 1 - g;                   // blob ring step
                if (issuer && st + AHEAD < G) issue(st + AHEAD);
                const int gs = gstep0 + st, stage = gs % S;
                mbar_wait(&bars[stage], uint32_t((gs / S) & 1));
                const double *blob = sblob + stage * BLOB;
                const double *tau = blob + KF * 2 * WP;
                const int c0 = (h + KP * r) % NPR;          // first v pair of this lane's slots
                // the window-aligned blob makes the reflector body independent of a: one copy of it
                // per rotation (the unrolled version missed the instruction cache, "no_instruction"
                // 3.4 stalls per issue)
#pragma unroll 1
                for (int a = 0; a < KF; a++) {
                    const double2 *v2 = reinterpret_cast<const double2 *>(blob + a * 2 * WP) + c0;
                    constexpr int LA = 8;                   // shared-memory loads in flight ahead of use
                    double2 vr[LA];
                    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                    for (int i = 0; i < LA && i < NL; i++) vr[i] = lds_v2(v2 + 2 * i);
#pragma unroll
                    for (int l = 0; l < NL; l++) {
                        const double2 vv = vr[l % LA];
                        if (l + LA < NL) vr[l % LA] = lds_v2(v2 + 2 * (l + LA));
                        acc[2 * (l & 1)] = fma(vv.x, qh[l].x, acc[2 * (l & 1)]);
                        acc[2 * (l & 1) + 1] = fma(vv.y, qh[l].y, acc[2 * (l & 1) + 1]);
                    }
                    double part = (acc[0] + acc[1]) + (acc[2] + acc[3]);
                    part += __shfl_xor_sync(0xffffffffu, part, 1);  // both halves of v^T q
                    const double w = -tau[a] * part;
#pragma unroll
                    for (int i = 0; i < LA && i < NL; i++) vr[i] = lds_v2(v2 + 2 * i);
#pragma unroll
                    for (int l = 0; l < NL; l++) {
                        const double2 vv = vr[l % LA];
                        if (l + LA < NL) vr[l % LA] = lds_v2(v2 + 2 * (l + LA));
                        qh[l].x = fma(vv.x, w, qh[l].x);
                        qh[l].y = fma(vv.y, w, qh[l].y);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&ebars[stage]);  // this warp is done with the stage
            }
            // emit the bottom KF rows (rows >= n do not exist; the warm-up emits nothing real)
            const int rb = top + WP - KF;
            if (rb < n) {
#pragma unroll
                for (int i = 0; i < KP; i++) {
                    const int s = slot(NPR - KP + i);
                    if ((s & 1) == h) st_pair(rb + 2 * i, qh[s >> 1]);
                }
            }
            const bool pub = t + 1 < T && ((pub_count == pub_period - 1) || (early && rb <= next_top0));
            if (pub && rb <= next_top0) early = false;
            if (pub) {
                __threadfence();
                __syncthreads();
                if (threadIdx.x == 0) st_release_u64(prog + k, uint64_t(n - min(rb, n)));
            }
            pub_count = pub ? 0 : pub_count + 1;
        };
        for (int t0 = 0; t0 < T; t0 += NW)
            dfma_static_for<0, NW>([&](auto rc) {
                const int t = t0 + decltype(rc)::value;
                if (t < T) step(rc, t);
            });
        __threadfence();
        __syncthreads();                                    // item complete
        if (threadIdx.x == 0) st_release_u64(prog + k, kPassDone);
        gstep0 += G;
    }
}

}  // namespace elpa_b200
