// kernel_dmma_kwin.cuh — a variant of the hot path (kernel_dmma.cuh) with
// one depth per work item and K reflector groups per step held in ONE register window of
// W = lambda + K - 1 chunks: group j of the step sits at chunk offset K-1-j, so the K groups of a
// step need no data movement between them, and the window slides by K chunks once per step
// (the FP32 kernel's window, kernel_f32.cuh, on the FP64 tensor cores).  Against the K = 1
// kernel this halves (K = 2) or quarters (K = 4) the register moves per group, and with 1-2 tiles
// per warp the window is small enough for 3-5 warps per SMSP.
//
// Step st of item (tile group x, depth m): window top chunk T(st) = C0 - st*K - (K-1); group-time
// tau = st*K + j applies group g = G-1-tau (top chunk C0 - tau = T(st) + K-1-j).  At the end of
// the step the bottom K chunks (T(st) + W-K ..) are final for depth m and go back to HBM, and the
// K chunks T(st+1) .. T(st+1) + K-1, prefetched with cp.async one step ahead, enter at the top.
// Work items, dequeue, the fragment ring (consumed mbarriers, no CTA barrier per step) and the
// progress words are those of kernel_dmma.cuh with D = 1, except that the words
// are per column warp (no CTA barrier on publish steps).
#pragma once
#include "kernel_dmma.cuh"


namespace elpa_b200 {

// Shared-memory and occupancy arithmetic of the kernel, also used by the host plan (make_plan).
constexpr int kwin_reg_est(int b8, int NCT, int K) { return 4 * (b8 + K) * NCT + 90; }   // W = b8 + K
constexpr int kwin_minb(int b8, int CW, int NCT, int K, int kind = KIND_DMMA) {
    // one-tile warps with two groups per step fit 128 registers without spills (118 at nbw = 64):
    // four CTAs of four warps per SM instead of three, +4-7% on thin stripes
    // (profiles/r02/kwin_nct1_minb4_r02.jsonl)
    const int reg = (kind == KIND_DMMA && NCT == 1 && K == 2) ? 128 : kwin_reg_est(b8, NCT, K);
    const int r = 65536 / (32 * CW * reg);
    return r < 1 ? 1 : (r > 8 ? 8 : r);
}
constexpr size_t kwin_smem(int b8, int CW, int NCT, int K, int stages, int kind = KIND_DMMA) {
    return size_t(stages) * K * (kind == KIND_ZMMA ? 256 : 128) * (b8 + 1) * 8   // ring: stages x K blobs
           + size_t(2) * K * CW * NCT * 64 * 8               // Q intake, double-buffered
           + size_t(2) * stages * 8 + 16;                    // mbarriers + item slot
}
// Fragment ring depth: 3 stages where they fit the register-limited CTA count (228 KB per SM, 1 KB
// reserved per CTA), else 2.  Measured at C3 (1,4,2,2): 2 -> 3 stages 30.42 -> 30.60 TF/s; a
// shape that would lose a CTA per SM keeps 2 ((1,2,2,2): 28.4 -> 23.7 with 3).
constexpr int kwin_stages(int b8, int CW, int NCT, int K, int kind = KIND_DMMA) {
    return size_t(kwin_minb(b8, CW, NCT, K, kind)) * (kwin_smem(b8, CW, NCT, K, 3, kind) + 1024) <= size_t(233472)
               ? 3 : 2;
}

// compile-time loop: f(integral_constant<int, I>) for I = I0 .. I1-1
template <int I0, int I1, class F>
__device__ __forceinline__ void static_for_kwin(F &&f) {
    if constexpr (I0 < I1) {
        f(std::integral_constant<int, I0>{});
        static_for_kwin<I0 + 1, I1>(f);
    }
}

// KIND_ZMMA: the complex Hermitian variant (NEXT-3), NCT real tiles = NCT/2 complex tiles as
// (Re, Im) pairs, ZmmaGroup's arithmetic (kernel_dmma.cuh) on the same window.
template <int B8, int CW, int NCT, int K, int KIND = KIND_DMMA>
struct KwinCfg {
    static constexpr int LAM = B8 + 1;
    static constexpr int ZF = (KIND == KIND_ZMMA) ? 2 : 1; // real tiles per (complex) tile
    static constexpr int W = LAM + K - 1;                 // window chunks
    static constexpr int BLOB = 128 * ZF * LAM;           // doubles per prepared group
    static constexpr int THREADS = 32 * CW;
    static constexpr int T = CW * NCT / ZF;               // 8-column tiles per work item
    static constexpr int STAGES = kwin_stages(B8, CW, NCT, K, KIND);   // fragment ring (K blobs per stage)
    static constexpr size_t SMEM_BLOBS = size_t(STAGES) * K * BLOB * sizeof(double);
    static constexpr size_t SMEM_INTAKE = size_t(2) * K * CW * NCT * 64 * sizeof(double);
    static constexpr size_t SMEM = kwin_smem(B8, CW, NCT, K, STAGES, KIND);
    static constexpr int MINB = kwin_minb(B8, CW, NCT, K, KIND);
};

// One compact-WY group (DmmaGroup's arithmetic) on window chunks [OFF, OFF + LAM) of q[NCT][W].
template <int LAM, int NCT, int W, int OFF>
__device__ __forceinline__ void dmma_group_at(double2 (&q)[NCT][W], const double *blob, int lane) {
    const double2 *dotB = reinterpret_cast<const double2 *>(blob);
    const double2 *updB = dotB + 32 * LAM;
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
            dmma(ya.x, ya.y, q[t][OFF + i].x, vb.x);
            dmma(yb.x, yb.y, q[t][OFF + i].y, vb.y);
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
#pragma unroll
    for (int i = 0; i < LAM; i++) {
        const double2 ub = updB[i * 32 + lane];
#pragma unroll
        for (int t = 0; t < NCT; t++) {
            dmma(q[t][OFF + i].x, q[t][OFF + i].y, w[t].x, ub.x);
            dmma(q[t][OFF + i].x, q[t][OFF + i].y, w[t].y, ub.y);
        }
    }
}

// One complex group (ZmmaGroup's arithmetic, kernel_dmma.cuh) on window chunks [OFF, OFF + LAM):
// q[2u] = Re, q[2u+1] = Im of complex tile u.
template <int LAM, int NCT, int W, int OFF>
__device__ __forceinline__ void zmma_group_at(double2 (&q)[NCT][W], const double *blob, int lane) {
    constexpr int NZ = NCT / 2;
    const double2 *dUr = reinterpret_cast<const double2 *>(blob);
    const double2 *dUi = dUr + 32 * LAM;
    const double2 *uVr = dUr + 64 * LAM;
    const double2 *uVi = dUr + 96 * LAM;
    double2 ya[NZ], yb[NZ], yc[NZ], yd[NZ];                // Qr.Ur, Qi.Ui, Qi.Ur, Qr.Ui
#pragma unroll
    for (int u = 0; u < NZ; u++) ya[u] = yb[u] = yc[u] = yd[u] = make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < LAM; i++) {
        const double2 ur = dUr[i * 32 + lane], ui = dUi[i * 32 + lane];
#pragma unroll
        for (int u = 0; u < NZ; u++) {
            const double2 qr = q[2 * u][OFF + i], qi = q[2 * u + 1][OFF + i];
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
            double2 &qr = q[2 * u][OFF + i];
            double2 &qi = q[2 * u + 1][OFF + i];
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

template <int KIND, int LAM, int NCT, int W, int OFF>
__device__ __forceinline__ void kwin_group_at(double2 (&q)[NCT][W], const double *blob, int lane) {
    if constexpr (KIND == KIND_ZMMA) zmma_group_at<LAM, NCT, W, OFF>(q, blob, lane);
    else dmma_group_at<LAM, NCT, W, OFF>(q, blob, lane);
}

template <int B8, int CW, int NCT, int K, int KIND = KIND_DMMA>
__global__ void __launch_bounds__(KwinCfg<B8, CW, NCT, K, KIND>::THREADS, KwinCfg<B8, CW, NCT, K, KIND>::MINB)
apply_dmma_kwin_kernel(int64_t n64, int64_t nev64, const double *__restrict__ blobs, double *Q, int64_t ldq,
                       uint64_t *prog, int pub_period) {
    using Cfg = KwinCfg<B8, CW, NCT, K, KIND>;
    constexpr int ZF = Cfg::ZF;
    constexpr int LAM = Cfg::LAM, W = Cfg::W, BLOB = Cfg::BLOB, S = Cfg::STAGES, T = Cfg::T;
    constexpr int B = 8 * B8;
    constexpr int AHEAD = S - 1;                           // the issuer waits only for its own last step

    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *sblob = reinterpret_cast<double *>(smem_raw);                                   // [S][K][BLOB]
    double2 *sintake = reinterpret_cast<double2 *>(smem_raw + Cfg::SMEM_BLOBS);             // [2][K][CW][NCT][32]
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + Cfg::SMEM_BLOBS + Cfg::SMEM_INTAKE);
    uint64_t *ebars = bars + S;
    int *s_item = reinterpret_cast<int *>(ebars + S);

    const int n = int(n64), nev = int(nev64);
    const int cw = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int M = int(num_depths(n64, B));
    const int C0 = (n - 2) >> 3;
    const int ntile = (nev + 7) >> 3;
    const int NX = (ntile + T - 1) / T;
    const int rsub = 2 * (lane & 3);
    constexpr uint32_t kAllTiles = (1u << NCT) - 1u;
    auto islot = [&](int par, int j, int t) { return (((par * K + j) * CW + cw) * NCT + t) * 32 + lane; };
    const bool issuer = threadIdx.x == 32 * (CW - 1);

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; i++) mbar_init(&bars[i], 1);
        for (int i = 0; i < S; i++) mbar_init(&ebars[i], CW);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    int gstep0 = 0;                                        // ring position of the item's step 0

    for (;;) {
        if (threadIdx.x == 0)
            *s_item = int(atomicAdd(reinterpret_cast<unsigned long long *>(prog + int64_t(NX) * M * CW), 1ull));
        __syncthreads();
        const int k = *s_item;
        if (k >= NX * M) break;
        const int p = k / NX, x = k % NX;                  // depth p, tile group x
        // progress word of this warp's columns in item k: column warp cw of item (x, p + 1) reads
        // exactly the columns column warp cw of item (x, p) writes, so each warp publishes its own
        // word (release after its lanes' fences) and waits on its producer warp's word only
        uint64_t *wprog = prog + int64_t(k) * CW + cw;
        const int tile_end = min(ntile, (x + 1) * T);
        double *qcol[NCT];
        uint32_t okmask = 0;
#pragma unroll
        for (int t = 0; t < NCT; t++) {
            const int tile = x * T + cw * (NCT / ZF) + t / ZF;
            const int c = tile * 8 + (lane >> 2);
            if (tile < tile_end && c < nev) okmask |= 1u << t;
            qcol[t] = Q + int64_t(ZF) * int64_t(min(c, nev - 1)) * ldq;
        }
        const int G = int(groups_at_depth(n64, B8, p));
        const int NT = G;                                  // group-times of this item
        const int nsteps = (NT + K - 1) / K;
        const double *bbase = blobs + group_base(n64, B8, p) * BLOB;

        int pub_count = 0;
        auto pub_step = [&](int st) {                      // cbot: lowest chunk final after step st
            const int cbot = C0 - st * K - (K - 1) + W - K;
            // every pub_period steps, and at the step whose emission first reaches chunk C0 (the
            // next depth's first window can start)
            return (pub_count == pub_period - 1 || (cbot <= C0 && cbot + K > C0)) && cbot <= C0 + 1 && cbot >= 0;
        };
        auto issue = [&](int st) {                         // fragments of step st -> ring stage
            const int gs = gstep0 + st, stg = gs % S;
            if (gs >= S) mbar_wait(&ebars[stg], uint32_t(((gs / S) - 1) & 1));
            uint32_t bytes = 0;
            for (int j = 0; j < K; j++)
                if (st * K + j < NT) bytes += BLOB * 8;
            mbar_arrive_expect_tx(&bars[stg], bytes);
            for (int j = 0; j < K; j++)
                if (st * K + j < NT)
                    bulk_g2s(sblob + (stg * K + j) * BLOB, bbase + int64_t(G - 1 - (st * K + j)) * BLOB, BLOB * 8,
                             &bars[stg]);
        };
        if (issuer)
            for (int st = 0; st < AHEAD && st < nsteps; st++) issue(st);

        uint32_t seen = 0;
        auto await_chunk = [&](int c) {                    // chunk c final from depth p-1
            if (p == 0 || c < 0) return;
            const uint32_t need = uint32_t(C0 + 2 - c);
            if (seen >= need) return;
            if (lane == 0) {
                uint64_t v = ld_acquire_u64(wprog - int64_t(NX) * CW);
                ELPA_WATCHDOG_START();
                while (v < need) {
                    __nanosleep(128);
                    v = ld_acquire_u64(wprog - int64_t(NX) * CW);
                    ELPA_WATCHDOG_CHECK();
                }
                seen = v > 0xFFFFFFFFull ? 0xFFFFFFFFu : uint32_t(v);
            }
            seen = __shfl_sync(0xffffffffu, seen, 0);
        };
        // the K chunks entering at the end of step st (window top of step st+1 = T(st) - K) -> slot st & 1
        auto intake = [&](int st) {
            const int top = C0 - (st + 1) * K - (K - 1);
            await_chunk(top);
#pragma unroll
            for (int j = 0; j < K; j++) {
                const int c = top + j;
                if constexpr (ZF == 2) {
#pragma unroll
                    for (int t = 0; t < NCT; t += 2)
                        zload_pair_async(&sintake[islot(st & 1, j, t)], &sintake[islot(st & 1, j, t + 1)], qcol[t],
                                         (okmask >> t) & 1, n, 8 * c + rsub);
                } else if (okmask == kAllTiles && c >= 0 && 8 * c + 8 <= n) {
#pragma unroll
                    for (int t = 0; t < NCT; t++)
                        cp_async16_zfill(&sintake[islot(st & 1, j, t)], qcol[t] + 8 * c + rsub, 16u);
                } else {
#pragma unroll
                    for (int t = 0; t < NCT; t++)
                        load_pair_async(&sintake[islot(st & 1, j, t)], qcol[t], (okmask >> t) & 1, n, 8 * c + rsub);
                }
            }
            cp_async_commit();
        };
        auto store_tiles = [&](const double2 *v, int r) {  // v[t], t < NCT
            if constexpr (ZF == 2) {
#pragma unroll
                for (int t = 0; t < NCT; t += 2) zstore_pair(qcol[t], (okmask >> t) & 1, n, r, v[t], v[t + 1]);
                return;
            }
            if (okmask == kAllTiles && r >= 0 && r + 2 <= n) {
#pragma unroll
                for (int t = 0; t < NCT; t++) *reinterpret_cast<double2 *>(qcol[t] + r) = v[t];
                return;
            }
#pragma unroll
            for (int t = 0; t < NCT; t++) store_pair(qcol[t], (okmask >> t) & 1, n, r, v[t]);
        };

        double2 q[NCT][W];
        const int T0 = C0 - (K - 1);
        await_chunk(T0);
#pragma unroll
        for (int i = 0; i < W; i++) {
            if constexpr (ZF == 2) {
#pragma unroll
                for (int t = 0; t < NCT; t += 2)
                    zload_pair(qcol[t], (okmask >> t) & 1, n, 8 * (T0 + i) + rsub, q[t][i], q[t + 1][i]);
            } else {
#pragma unroll
                for (int t = 0; t < NCT; t++) q[t][i] = load_pair(qcol[t], (okmask >> t) & 1, n, 8 * (T0 + i) + rsub);
            }
        }
        if (nsteps > 1) intake(0);

        int st = 0;
        for (;; st++) {
            if (issuer && st + AHEAD < nsteps) issue(st + AHEAD);
            if (st + 1 < nsteps - 1) intake(st + 1);       // chunks entering at the end of step st + 1
            const int gs = gstep0 + st, stage = gs % S;
            mbar_wait(&bars[stage], uint32_t((gs / S) & 1));
            const double *sb = sblob + stage * K * BLOB;
            if (st * K + K <= NT) {                        // a full step: one basic block, so the
                static_for_kwin<0, K>([&](auto jc) {       // groups' DMMAs interleave (+1.7% at C3)
                    constexpr int j = decltype(jc)::value;
                    kwin_group_at<KIND, LAM, NCT, W, K - 1 - j>(q, sb + j * BLOB, lane);
                });
            } else {                                       // the item's last step, NT % K groups
                static_for_kwin<0, K>([&](auto jc) {
                    constexpr int j = decltype(jc)::value;
                    if (st * K + j < NT) kwin_group_at<KIND, LAM, NCT, W, K - 1 - j>(q, sb + j * BLOB, lane);
                });
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&ebars[stage]);     // this warp is done with the stage
            if (st + 1 >= nsteps) break;                   // the final window is written back below
            // emit the bottom K chunks: final for this depth
            const int tst = C0 - st * K - (K - 1);
#pragma unroll
            for (int jj = 0; jj < K; jj++) {
                double2 bot[NCT];
#pragma unroll
                for (int t = 0; t < NCT; t++) bot[t] = q[t][W - K + jj];
                store_tiles(bot, 8 * (tst + W - K + jj) + rsub);
            }
            const bool pub = pub_step(st);
            if (pub) __threadfence();                      // this lane's stores, before the warp's release
            // slide by K chunks; the new top chunks arrived during this step
            if (st + 1 < nsteps - 1) cp_async_wait<1>(); else cp_async_wait<0>();
#pragma unroll
            for (int t = 0; t < NCT; t++) {
#pragma unroll
                for (int i = W - 1; i >= K; i--) q[t][i] = q[t][i - K];
                if constexpr (ZF == 2) {
                    if (t & 1) {                           // the (Re, Im) pair, split at its odd member
#pragma unroll
                        for (int j = 0; j < K; j++)
                            zsplit(sintake[islot(st & 1, j, t - 1)], sintake[islot(st & 1, j, t)], q[t - 1][j], q[t][j]);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < K; j++) q[t][j] = sintake[islot(st & 1, j, t)];
                }
            }
            if (pub) {                                     // per-warp word: no CTA barrier
                __syncwarp();
                if (lane == 0) st_release_u64(wprog, uint64_t(C0 + 2 - (tst + W - K)));
            }
            pub_count = pub ? 0 : pub_count + 1;
        }
        cp_async_wait<0>();
        // write back the final window: top chunk T(st)
        const int tf = C0 - st * K - (K - 1);
#pragma unroll
        for (int i = 0; i < W; i++) {
            double2 col[NCT];
#pragma unroll
            for (int t = 0; t < NCT; t++) col[t] = q[t][i];
            store_tiles(col, 8 * (tf + i) + rsub);
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release_u64(wprog, kPassDone);  // this warp's columns of the pass are final
        __syncthreads();                                   // s_item is rewritten by the next dequeue
        gstep0 += nsteps;
    }
}

}  // namespace elpa_b200
