// kernel_f32.cuh — NEXT-3: the single-precision variant of the hot path.  ELPA
// runs the whole two-stage solver in FP32 as well, and single precision in the
// eigen-steps is where the paper's mixed-precision speed-ups come from.
//
// Same operation as the FP64 path, on FP32 data:  Q <- H_0 H_1 ... H_{R-1} Q  (H_{R-1} first).
// Same schedule: work items (column block, depth pass), k = 8 sweep groups per depth in
// group-time order, D depth warps stacked with the shared-memory hand-off, cross-pass
// progress words (kernel_dmma.cuh).  The arithmetic is different:
//   * there is no FP32 tensor-core MMA (TF32 rounds the operands to 10 mantissa bits), so
//     the group runs on the FP32 pipe, and the packed fma.rn.f32x2 (SASS FFMA2, sm_100)
//     does two FMAs per lane per instruction;
//   * a lane owns whole columns (NC of them, 32*NC columns per warp) with the b+8-row window
//     in registers as row PAIRS (f2 = {row 2p, row 2p+1}), so the dot products need no
//     shuffles and the reflector vectors are warp-broadcast shared-memory reads;
//   * reflectors are applied one at a time in exact generation order inside the group (no
//     compact-WY factor, no padding flops: a = 0..7, each w = tau v^T q then q -= w v),
//     i.e. the plain Householder recurrence the oracle follows, in FP32 with FMA.
// Blob (per group, prep_f32_kernel): reflector a's vector laid out as row pairs starting at
// pair p0(a) = (7-a)/2 of the window, VP = 4*b8 + 2 pairs each (zeros outside [7-a, 7-a+L)),
// then tau[8].
#pragma once
#include "kernel_dmma.cuh"

namespace elpa_b200 {

typedef unsigned long long f2_t;   // two FP32 values: low half = even row, high half = odd row

__device__ __forceinline__ f2_t ffma2(f2_t a, f2_t b, f2_t c) {
    f2_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2_t fadd2(f2_t a, f2_t b) {
    f2_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ float f2_lo(f2_t x) { return __uint_as_float(uint32_t(x)); }
__device__ __forceinline__ float f2_hi(f2_t x) { return __uint_as_float(uint32_t(x >> 32)); }
__device__ __forceinline__ f2_t f2_splat(float w) {
    const f2_t u = __float_as_uint(w);
    return u | (u << 32);
}
__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
    return f2_t(__float_as_uint(lo)) | (f2_t(__float_as_uint(hi)) << 32);
}

// floats per prepared FP32 group: 8 reflectors x VP pairs x 2, then tau[8]
__host__ __device__ constexpr int f32_vp(int b8) { return 4 * b8 + 2; }
__host__ __device__ constexpr int64_t f32_blob_floats(int b8) { return 16 * f32_vp(b8) + 8; }

#ifndef F32_VBARRIER
#define F32_VBARRIER() asm volatile("" ::: "memory")
#endif
// One FP32 group for one warp: NC columns per lane, window q[t][pair] (NPW = 4*lambda pairs).
template <int B8, int NC>
struct F32Group {
    static constexpr int LAM = B8 + 1;
    static constexpr int NPW = 4 * LAM;
    static constexpr int VP = f32_vp(B8);
    static constexpr int NPAIR = 4 * B8 + 1;     // pairs a reflector spans (b rows, start parity)
    static constexpr int BLOB = int(f32_blob_floats(B8));
    // applies the group to window pairs [OFF, OFF + NPW) of a register window of NW pairs
    template <int OFF, int NW>
    __device__ __forceinline__ static void apply(f2_t (&q)[NC][NW], const float *blob) {
        const ulonglong2 *vb = reinterpret_cast<const ulonglong2 *>(blob);
        const float *tau = blob + 16 * VP;
#pragma unroll
        for (int a = 0; a < 8; a++) {
            const int p0 = OFF + ((7 - a) >> 1);
            const ulonglong2 *v = vb + a * (VP / 2);
            // w = tau * v^T q: two accumulators per column (even / odd pair index)
            f2_t acc[NC][2];
#pragma unroll
            for (int t = 0; t < NC; t++) acc[t][0] = acc[t][1] = 0ull;
#pragma unroll
            for (int k2 = 0; k2 < VP / 2; k2++) {
                const ulonglong2 vv = v[k2];
                F32_VBARRIER();
#pragma unroll
                for (int t = 0; t < NC; t++) {
                    acc[t][0] = ffma2(q[t][p0 + 2 * k2], vv.x, acc[t][0]);
                    if (2 * k2 + 1 < NPAIR) acc[t][1] = ffma2(q[t][p0 + 2 * k2 + 1], vv.y, acc[t][1]);
                }
            }
            const float ta = tau[a];
            f2_t w2[NC];
#pragma unroll
            for (int t = 0; t < NC; t++) {
                const f2_t s2 = fadd2(acc[t][0], acc[t][1]);
                w2[t] = f2_splat(-ta * (f2_lo(s2) + f2_hi(s2)));
            }
            // q -= w v (v is re-read from shared memory: keeping the b floats of v live from the
            // dot would cost b registers on top of the window)
            asm volatile("" ::: "memory");
#pragma unroll
            for (int k2 = 0; k2 < VP / 2; k2++) {
                const ulonglong2 vv = v[k2];
                F32_VBARRIER();
#pragma unroll
                for (int t = 0; t < NC; t++) {
                    q[t][p0 + 2 * k2] = ffma2(vv.x, w2[t], q[t][p0 + 2 * k2]);
                    if (2 * k2 + 1 < NPAIR) q[t][p0 + 2 * k2 + 1] = ffma2(vv.y, w2[t], q[t][p0 + 2 * k2 + 1]);
                }
            }
        }
    }
};

// Reflector preparation: one warp per group (m, g); sweeps j = 8g+6-a, reflector a starts at
// window row 7-a; missing reflectors (j < 0 or j > J_m) are zero with tau = 0.
template <int B8>
__global__ void __launch_bounds__(256)
prep_f32_kernel(int64_t n, const float *__restrict__ hh_v, const float *__restrict__ hh_tau,
                float *__restrict__ blobs) {
    constexpr int B = 8 * B8;
    constexpr int VP = f32_vp(B8);
    constexpr int BLOB = int(f32_blob_floats(B8));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t m = blockIdx.y;
    const int64_t g = (int64_t)blockIdx.x * 8 + warp;
    if (g >= groups_at_depth(n, B8, m)) return;
    const int64_t Jm = n - 3 - m * B;
    float *blob = blobs + (group_base(n, B8, m) + g) * BLOB;
    for (int e = lane; e < 16 * VP; e += 32) {
        const int a = e / (2 * VP), w = e % (2 * VP);
        const int row = 2 * ((7 - a) >> 1) + w;          // window row of this element
        const int i = row - (7 - a);                      // index into the reflector's vector
        const int64_t j = 8 * g + 6 - a;
        float val = 0.0f;
        if (j >= 0 && j <= Jm && i >= 0) {
            const int64_t s = j + 1 + m * B;
            const int64_t L = (n - s < B) ? (n - s) : B;
            if (i < L) val = (i == 0) ? 1.0f : hh_v[(hh_off(j, n, B) + m) * B + i];
        }
        blob[e] = val;
    }
    if (lane < 8) {
        const int64_t j = 8 * g + 6 - lane;
        blob[16 * VP + lane] = (j >= 0 && j <= Jm) ? hh_tau[hh_off(j, n, B) + m] : 0.0f;
    }
}

// FP32 chunk I/O: lane's 8 rows [8c, 8c+8) of one column = 4 pairs; rows outside [0, n) read
// as zero and are never written; masked-off columns likewise.
__device__ __forceinline__ void f32_load_chunk(f2_t *dst, const float *colp, bool ok, int n, int c) {
    const int r = 8 * c;
    if (ok && r >= 0 && r + 8 <= n) {
        const ulonglong2 a = *reinterpret_cast<const ulonglong2 *>(colp + r);
        const ulonglong2 b = *reinterpret_cast<const ulonglong2 *>(colp + r + 4);
        dst[0] = a.x; dst[1] = a.y; dst[2] = b.x; dst[3] = b.y;
        return;
    }
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; i++) v[i] = (ok && r + i >= 0 && r + i < n) ? colp[r + i] : 0.0f;
#pragma unroll
    for (int i = 0; i < 4; i++) dst[i] = f2_pack(v[2 * i], v[2 * i + 1]);
}
__device__ __forceinline__ void f32_load_chunk_async(ulonglong2 *d0, ulonglong2 *d1, const float *colp, bool ok,
                                                     int n, int c) {
    const int r = 8 * c;
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int rh = r + 4 * h;
        int rem = (ok && rh >= 0) ? n - rh : 0;
        rem = rem < 0 ? 0 : (rem > 4 ? 4 : rem);
        cp_async16_zfill(h ? d1 : d0, rem ? colp + rh : colp, uint32_t(rem * 4));
    }
}
__device__ __forceinline__ void f32_store_chunk(float *colp, bool ok, int n, int c, const f2_t *src) {
    const int r = 8 * c;
    if (!ok || r < 0) return;
    if (r + 8 <= n) {
        *reinterpret_cast<ulonglong2 *>(colp + r) = make_ulonglong2(src[0], src[1]);
        *reinterpret_cast<ulonglong2 *>(colp + r + 4) = make_ulonglong2(src[2], src[3]);
        return;
    }
#pragma unroll
    for (int i = 0; i < 8; i++)
        if (r + i < n) colp[r + i] = (i & 1) ? f2_hi(src[i >> 1]) : f2_lo(src[i >> 1]);
}

// compile-time loop: f(integral_constant<int, I>) for I = I0 .. I1-1
template <int I0, int I1, class F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr (I0 < I1) {
        f(std::integral_constant<int, I0>{});
        static_for<I0 + 1, I1>(f);
    }
}

template <int B8, int D, int CW, int NC, int K>
struct F32Cfg {
    static constexpr int LAM = B8 + 1;
    using Group = F32Group<B8, NC>;
    static constexpr int BLOB = Group::BLOB;                // floats per prepared group
    static constexpr int W = LAM + K - 1;                  // register window in chunks
    static constexpr int NWP = 4 * W;                      // ... in row pairs
    static constexpr int NWARP = D * CW;
    static constexpr int THREADS = 32 * NWARP;
    static constexpr int COLS = CW * NC * 32;              // columns per work item
    static constexpr int STAGES = (K * D * BLOB * 4 * 3 <= 100 * 1024) ? 3 : 2;
    // shared memory: STAGES x K x D blobs, hand-off chunks [2][D][K][CW][NC][2][32] x 16 B,
    // warp-0 intake chunks [2][K][CW][NC][2][32] x 16 B, barriers + the dequeued item index
    static constexpr size_t SMEM_BLOBS = size_t(STAGES) * K * D * BLOB * sizeof(float);
    static constexpr size_t SMEM_HAND = size_t(2) * D * K * CW * NC * 2 * 32 * 16;
    static constexpr size_t SMEM_INTAKE = size_t(2) * K * CW * NC * 2 * 32 * 16;
    static constexpr size_t SMEM = SMEM_BLOBS + SMEM_HAND + SMEM_INTAKE + 64;
    // Register cap (__maxnreg__): the window is 8*W*NC floats.  NC = 1, K = 1 at nbw <= 64
    // compiles without spills in 168 (6 CTAs of 64 threads per SM); larger windows get 255.
    // (A minBlocks launch bound instead spills at the same count.)
    static constexpr int REGCAP = (NC == 1 && K == 1 && B8 <= 8) ? 168 : 255;
};

// The persistent item kernel of kernel_dmma.cuh (work items, dynamic dequeue, progress words:
// DESIGN.md §5) with FP32 windows, F32Group arithmetic and K groups per step.
//
// Step st of an item applies group-times tau = st*K + j, j = 0..K-1: depth warp d applies
// group g = G - 1 - tau + d*K of depth m0 + d.  Its register window holds W = lambda + K - 1
// chunks, top chunk T_d(st) = C0 - st*K - (K-1) + d*W, so group j sits at chunk offset
// K-1-j and the K groups of a step need no data movement between them.  The D windows are
// stacked without gaps and without chunks in transit: at the end of a step every warp emits
// its bottom K chunks (to HBM from the deepest warp, else to warp d+1 through shared memory);
// at the start of the next step it shifts its window down by K chunks and takes in K new top
// chunks (HBM for warp 0, prefetched with cp.async one step ahead).  Depth m0+d+1 thus trails
// depth m0+d by K groups, one step: the schedule legality of DESIGN.md §5 (a reflector of
// depth m+1 overlaps only reflectors of depth m with a larger sweep index, all in groups
// with index >= its own) holds with one barrier per step.  Register moves: 4*(W-K) pairs per
// step, i.e. 4*(lambda-1)/K per group.
template <int B8, int D, int CW, int NC, int K>
__global__ void __maxnreg__((F32Cfg<B8, D, CW, NC, K>::REGCAP))
apply_f32_kernel(int64_t n64, int64_t nev64, const float *__restrict__ blobs, float *Q, int64_t ldq,
                 uint64_t *prog, int pub_period) {
    using Cfg = F32Cfg<B8, D, CW, NC, K>;
    using Group = typename Cfg::Group;
    constexpr int W = Cfg::W;
    constexpr int NWP = Cfg::NWP;
    constexpr int BLOB = Cfg::BLOB;
    constexpr int S = Cfg::STAGES;
    constexpr int COLS = Cfg::COLS;
    constexpr int B = 8 * B8;
    constexpr int LAG = K;                                 // groups depth m+1 trails depth m
    constexpr int SPAN = W;                                // chunk distance between stacked windows

    extern __shared__ __align__(128) unsigned char smem_raw[];
    float *sblob = reinterpret_cast<float *>(smem_raw);                                              // [S][K][D][BLOB]
    ulonglong2 *shand = reinterpret_cast<ulonglong2 *>(smem_raw + Cfg::SMEM_BLOBS);
    ulonglong2 *sintake = reinterpret_cast<ulonglong2 *>(smem_raw + Cfg::SMEM_BLOBS + Cfg::SMEM_HAND);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + Cfg::SMEM_BLOBS + Cfg::SMEM_HAND + Cfg::SMEM_INTAKE);
    int *s_item = reinterpret_cast<int *>(bars + S);

    const int n = int(n64), nev = int(nev64);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int d = warp / CW, cw = warp % CW;
    const int M = int(num_depths(n64, B));
    const int C0 = (n - 2) >> 3;
    const int NX = (nev + COLS - 1) / COLS;
    const int NP = (M + D - 1) / D;
    // hand-off slot (parity, receiving depth, chunk j of the step, column t, half h) / intake slot
    auto hslot = [&](int par, int dd, int j, int t, int h) {
        return (((((par * D + dd) * K + j) * CW + cw) * NC + t) * 2 + h) * 32 + lane;
    };
    auto islot = [&](int par, int j, int t, int h) {
        return ((((par * K + j) * CW + cw) * NC + t) * 2 + h) * 32 + lane;
    };
    // the blob ring is fed by one thread of the deepest depth row (no intake work there)
    const bool issuer = threadIdx.x == 32 * (D - 1) * CW;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; i++) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    uint32_t phase_bits = 0;
    int stage0 = 0;

    for (;;) {
        if (threadIdx.x == 0)
            *s_item = int(atomicAdd(reinterpret_cast<unsigned long long *>(prog + int64_t(NX) * NP), 1ull));
        __syncthreads();
        const int k = *s_item;
        if (k >= NX * NP) break;
        const int p = k / NX, x = k % NX;
        const int m0 = p * D;
        float *qcol[NC];
        uint32_t okmask = 0;
#pragma unroll
        for (int t = 0; t < NC; t++) {
            const int c = x * COLS + (cw * NC + t) * 32 + lane;
            if (c < nev) okmask |= 1u << t;
            qcol[t] = Q + int64_t(min(c, nev - 1)) * ldq;
        }
        const int G = int(groups_at_depth(n64, B8, m0));
        const int dmax = min(D, M - m0) - 1;
        const int NT = G + dmax * LAG;                     // group-times of this item
        const int nsteps = (NT + K - 1) / K;
        const int T0 = C0 - (K - 1) + d * SPAN;            // this warp's window top at step 0

        // deepest warps' lowest emitted chunk after step st; chunks >= it are final
        auto deep_cbot = [&](int st) { return C0 - st * K - (K - 1) + (D - 1) * SPAN + W - K; };
        int pub_count = 0;
        auto pub_step = [&](int st) {
            const int cbot = deep_cbot(st);
            return (pub_count == pub_period - 1 || cbot == C0) && cbot <= C0 + 1 && cbot >= 0;
        };
        auto group_valid = [&](int tau, int dd) {
            const int g = G - 1 - tau + dd * LAG;
            return dd <= dmax && tau < NT && g >= 0 && g < G - dd * B8;
        };
        auto issue = [&](int st) {                         // K x D blobs of step st -> ring stage
            const int stg = (stage0 + st) % S;
            uint64_t *bar = &bars[stg];
            uint32_t bytes = 0;
            for (int j = 0; j < K; j++)
                for (int dd = 0; dd <= dmax; dd++)
                    if (group_valid(st * K + j, dd)) bytes += BLOB * 4;
            mbar_arrive_expect_tx(bar, bytes);
            for (int j = 0; j < K; j++)
                for (int dd = 0; dd <= dmax; dd++)
                    if (group_valid(st * K + j, dd)) {
                        const int g = G - 1 - (st * K + j) + dd * LAG;
                        const float *src = blobs + (group_base(n64, B8, m0 + dd) + g) * BLOB;
                        bulk_g2s(sblob + ((stg * K + j) * D + dd) * BLOB, src, BLOB * 4, bar);
                    }
        };
        if (issuer)
            for (int st = 0; st < S - 1 && st < nsteps; st++) issue(st);

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
        // warp-0 intake of the K top chunks of step st (chunks T_0(st) + j), one step ahead
        auto intake = [&](int st) {
            const int top = T0 - st * K;
            await_chunk(top);
#pragma unroll
            for (int j = 0; j < K; j++)
#pragma unroll
                for (int t = 0; t < NC; t++)
                    f32_load_chunk_async(&sintake[islot(st & 1, j, t, 0)], &sintake[islot(st & 1, j, t, 1)], qcol[t],
                                         (okmask >> t) & 1, n, top + j);
            cp_async_commit();
        };

        f2_t q[NC][NWP];
        if (d == 0) await_chunk(T0);
#pragma unroll
        for (int t = 0; t < NC; t++)
#pragma unroll
            for (int i = 0; i < W; i++)
                f32_load_chunk(&q[t][4 * i], qcol[t], (okmask >> t) & 1, n, T0 + i);
        if (d == 0 && nsteps > 1) intake(1);

        for (int st = 0;; st++) {
            if (st > 0) {
                // take in the K new top chunks: shift the window down by K chunks
                if (d == 0) {
                    if (st + 1 < nsteps) intake(st + 1);
                    if (st + 1 < nsteps) cp_async_wait<1>(); else cp_async_wait<0>();
                }
#pragma unroll
                for (int t = 0; t < NC; t++) {
#pragma unroll
                    for (int i = NWP - 1; i >= 4 * K; i--) q[t][i] = q[t][i - 4 * K];
#pragma unroll
                    for (int j = 0; j < K; j++) {
                        const ulonglong2 lo2 = (d == 0) ? sintake[islot(st & 1, j, t, 0)]
                                                        : shand[hslot((st - 1) & 1, d, j, t, 0)];
                        const ulonglong2 hi2 = (d == 0) ? sintake[islot(st & 1, j, t, 1)]
                                                        : shand[hslot((st - 1) & 1, d, j, t, 1)];
                        q[t][4 * j] = lo2.x; q[t][4 * j + 1] = lo2.y; q[t][4 * j + 2] = hi2.x; q[t][4 * j + 3] = hi2.y;
                    }
                }
            }
            if (issuer && st + S - 1 < nsteps) issue(st + S - 1);
            const uint32_t stage = uint32_t((stage0 + st) % S);
            const uint32_t par = (phase_bits >> stage) & 1u;
            phase_bits ^= (1u << stage);
            bool waited = false;
            static_for<0, K>([&](auto jc) {
                constexpr int j = decltype(jc)::value;
                if (group_valid(st * K + j, d)) {
                    if (!waited) { mbar_wait(&bars[stage], par); waited = true; }
                    Group::template apply<4 * (K - 1 - j), NWP>(q, sblob + ((stage * K + j) * D + d) * BLOB);
                }
            });
            if (st + 1 >= nsteps) break;                   // final windows written back below
            // emit the bottom K chunks (window chunks W-K .. W-1 = T_d + W - K + jj)
            const int cb = T0 - st * K + W - K;
            if (d == D - 1) {
#pragma unroll
                for (int jj = 0; jj < K; jj++)
#pragma unroll
                    for (int t = 0; t < NC; t++)
                        f32_store_chunk(qcol[t], (okmask >> t) & 1, n, cb + jj, &q[t][4 * (W - K + jj)]);
                if (pub_step(st)) __threadfence();
            } else {
#pragma unroll
                for (int jj = 0; jj < K; jj++)
#pragma unroll
                    for (int t = 0; t < NC; t++) {
                        shand[hslot(st & 1, d + 1, jj, t, 0)] =
                            make_ulonglong2(q[t][4 * (W - K + jj)], q[t][4 * (W - K + jj) + 1]);
                        shand[hslot(st & 1, d + 1, jj, t, 1)] =
                            make_ulonglong2(q[t][4 * (W - K + jj) + 2], q[t][4 * (W - K + jj) + 3]);
                    }
            }
            __syncthreads();
            if (threadIdx.x == 0 && pub_step(st)) st_release_u64(prog + k, uint64_t(C0 + 2 - deep_cbot(st)));
            pub_count = (pub_count == pub_period - 1) ? 0 : pub_count + 1;
        }
        if (d == 0) cp_async_wait<0>();
        // write back the final windows (no chunks are in transit between windows)
        const int tf = T0 - (nsteps - 1) * K;
#pragma unroll
        for (int t = 0; t < NC; t++)
#pragma unroll
            for (int i = 0; i < W; i++)
                f32_store_chunk(qcol[t], (okmask >> t) & 1, n, tf + i, &q[t][4 * i]);
        __threadfence();
        __syncthreads();  // item complete: publish, and the smem ring/hand-off are free again
        if (threadIdx.x == 0) st_release_u64(prog + k, kPassDone);
        stage0 = (stage0 + nsteps) % S;
    }
}

// One thread per column, exact reverse generation order, explicitly rounded FP32 products and
// sums (the FP32 analogue of apply_reference_kernel; any nbw).
__global__ void __launch_bounds__(128)
apply_reference_f32_kernel(int64_t n, int64_t b, int64_t nev, const float *__restrict__ hh_v,
                           const float *__restrict__ hh_tau, float *Q, int64_t ldq) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nev) return;
    float *q = Q + c * ldq;
    for (int64_t j = n - 3; j >= 0; j--) {
        int64_t Mj = (n - 3 - j) / b + 1;
        int64_t off = hh_off(j, n, b);
        for (int64_t m = Mj - 1; m >= 0; m--) {
            int64_t r = off + m;
            int64_t s = j + 1 + m * b;
            int64_t L = (n - s < b) ? (n - s) : b;
            const float *v = hh_v + r * b;
            float sum = q[s];
            for (int64_t i = 1; i < L; i++) sum = __fadd_rn(sum, __fmul_rn(v[i], q[s + i]));
            float w = __fmul_rn(hh_tau[r], sum);
            q[s] = __fsub_rn(q[s], w);
            for (int64_t i = 1; i < L; i++) q[s + i] = __fsub_rn(q[s + i], __fmul_rn(w, v[i]));
        }
    }
}

}  // namespace elpa_b200
