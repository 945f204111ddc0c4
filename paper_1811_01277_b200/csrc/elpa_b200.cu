// elpa_b200.cu — C-ABI host library (include/elpa_b200.h): validation, closed-form
// reflector geometry, workspace handling and launch configuration for the sm_100a kernels.
// Build: see paper_1811_01277_b200/build.py (nvcc -gencode arch=compute_100a,code=sm_100a).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/elpa_b200.h"
#include "host_common.h"
#include "geometry.cuh"
#include "kernel_dmma.cuh"
#include "kernel_prep.cuh"
#include "kernel_dfma.cuh"
#include "kernel_dmma_kwin.cuh"
#include "kernel_reference.cuh"

#include <mutex>

using namespace elpa_b200;
using namespace elpa_b200_host;

namespace {

struct Plan {
    int kernel = ELPA_B200_KERNEL_REFERENCE;
    int b8 = 0, D = 1, CW = 1, NCT = 1, K = 1;
    int64_t nbw = 0;
    int kf = 0;                // DFMA kernel: reflectors fused per group (2, 4, 6, 8)
    int64_t gb_off = 0;        // DFMA kernel: byte offset of the group-base table in the workspace
    int grid_req = 0;          // requested grid (0 = co-resident maximum)
    int64_t items = 0;         // (tile group, depth pass) work items
    int64_t nx = 0;            // tile groups
    int64_t grid = 1;
    int threads = 128;
    size_t smem = 0;
    int64_t ws_bytes = 0;
};

// nbw = 8*b8 with b8 in 1..16 runs on the DMMA path; {1,2,4,8} (nbw 8/16/32/64) get the full
// shape menu, the other multiples of 8 up to 128 a small one (compile-time budget)
bool b8_full_menu(int b8) { return b8 == 1 || b8 == 2 || b8 == 4 || b8 == 8; }
bool b8_supported(int64_t nbw) { return nbw % 8 == 0 && nbw >= 8 && nbw <= 128; }

// (D, CW, NCT) menu of compiled DMMA configurations
// (D depth warps, CW column warps, NCT tiles per warp, K groups per step)
struct Shape { int D, CW, NCT, K; };
// K = 1 throughout for apply_dmma_kernel (its K = 2/4 variants were slower at every config,
// profiles/shape_sweep_r01_k.jsonl); groups_per_step K >= 2 selects the register-window kernel
// (kernel_dmma_kwin.cuh, kKwinShapes below).
#define ELPA_SHAPES(X) X(1, 2, 4, 1) X(2, 2, 4, 1) X(4, 2, 4, 1) X(8, 1, 4, 1) X(2, 4, 2, 1) X(2, 2, 3, 1) \
    X(2, 2, 2, 1) X(4, 4, 2, 1) X(2, 4, 3, 1) X(2, 1, 2, 1) X(1, 2, 2, 1) X(4, 2, 2, 1) X(2, 1, 4, 1) \
    X(1, 1, 4, 1) X(1, 1, 2, 1) X(1, 4, 2, 1) X(2, 1, 3, 1)
#define ELPA_SHAPE_ENTRY(D_, CW_, NCT_, K_) {D_, CW_, NCT_, K_},
constexpr Shape kShapes[] = {ELPA_SHAPES(ELPA_SHAPE_ENTRY)};

// The DFMA kernel (kernel_dfma.cuh) is compiled for nbw = 8/16/32/64, fused
// group sizes k = 2/4/6/8 and CW = 2 warps (64 columns) per CTA.
bool dfma_compiled(int64_t nbw, int kf, int CW) {
    return (nbw == 8 || nbw == 16 || nbw == 32 || nbw == 64) && (kf == 2 || kf == 4 || kf == 6 || kf == 8) && CW == 2;
}

#define ELPA_SMALL_SHAPES(X) X(2, 2, 2, 1) X(1, 2, 2, 1)
constexpr Shape kSmallShapes[] = {ELPA_SMALL_SHAPES(ELPA_SHAPE_ENTRY)};

// One depth per item and K >= 2 groups per step in one register window (kernel_dmma_kwin.cuh),
// compiled for nbw = 32 and 64: (1, CW, NCT, K)
#define ELPA_KWIN_SHAPES(X) X(1, 2, 2, 2) X(1, 4, 2, 2) X(1, 4, 1, 4) X(1, 4, 1, 2) X(1, 6, 2, 2) X(1, 8, 2, 2) \
    X(1, 3, 2, 2) X(1, 4, 2, 3) X(1, 8, 1, 2)
constexpr Shape kKwinShapes[] = {ELPA_KWIN_SHAPES(ELPA_SHAPE_ENTRY)};
bool kwin_compiled(int b8, int D, int CW, int NCT, int K) {
    if (b8 != 4 && b8 != 8) return false;
    for (const Shape &s : kKwinShapes)
        if (s.D == D && s.CW == CW && s.NCT == NCT && s.K == K) return true;
    return false;
}

bool shape_compiled(int D, int CW, int NCT, int K);
bool shape_compiled(int D, int CW, int NCT, int K, int b8) {
    if (!b8_full_menu(b8)) {
        for (const Shape &s : kSmallShapes)
            if (s.D == D && s.CW == CW && s.NCT == NCT && s.K == K) return true;
        return false;
    }
    return shape_compiled(D, CW, NCT, K);
}

bool shape_compiled(int D, int CW, int NCT, int K) {
    for (const Shape &s : kShapes)
        if (s.D == D && s.CW == CW && s.NCT == NCT && s.K == K) return true;
    return false;
}

size_t dmma_smem(int b8, int D, int CW, int NCT, int K) {
    const size_t blob = size_t(blob_doubles(b8 + 1, 0));
    const int stages = (K * D * blob * 8 * 3 <= 100 * 1024) ? 3 : 2;
    return size_t(stages) * K * D * blob * 8 + size_t(2) * D * K * CW * NCT * 64 * 8 +
           size_t(2) * K * CW * NCT * 64 * 8 + 64;
}

// DFMA workspace: the prepared groups, then the group-base table (M + 1 int64)
int64_t dfma_total_groups(int64_t n, int64_t nbw, int kf) {
    const int64_t M = num_depths(n, nbw);
    int64_t t = 0;
    for (int64_t m = 0; m < M; m++) t += dfma_groups(n, nbw, kf, m);
    return t;
}

// Automatic choice (measured sweeps in profiles/shape_sweep_r01*.jsonl):
// small CTAs (64-256 threads, 30-70 KB shared memory) so several share an SM and hide each
// other's per-step barriers; work items (tile group, depth pass) are spread dynamically over
// all SMs, so balance no longer depends on nev / (8 * #SMs).
void auto_shape(int64_t ntile, int64_t M, int b8, int &D, int &CW, int &NCT, int &K) {
    K = 1;
    // best of 5 per shape (profiles/shape_sweep_r01_final2.jsonl), TF/s:
    //                 C2    C4    C3/8  C3/4  C3    C5/8
    //   (1,2,4,1)   17.8  24.8  25.8  27.1  28.1  27.7
    //   (2,2,2,1)   19.4  25.7  26.6  27.4  27.7  27.5
    // MEDIUM autotuning with the final kernel (profiles/autotune_medium_r01_final.jsonl): C3 keeps
    // (1,2,4,1) 28.7, C4 keeps (2,2,2,1) 26.1, C2 (nbw = 32) prefers (4,2,2,1) 22.3 over 21.2
    // Round 2: nbw = 64 runs the two-group register window (kernel_dmma_kwin.cuh) everywhere
    // (profiles/r02/kwin_final_shapes_r02.jsonl, TF/s):
    //   columns (n = 20000)  500   1000  2000  2500  5000  10000 20000 | n = 60000: 3750  7500
    //   (1,4,2,2) K=2       14.2  22.7  26.7  27.1  29.0  29.9  30.6  |            28.4  29.0
    //   (1,4,1,2) K=2       21.6  24.7  26.5  26.6  27.2  27.3        |            26.4  26.5
    //   round 1's K = 1     19.7  24.3  26.7  27.0  28.1  28.6  29.0  |            27.4  27.9
    // With four CTAs per SM at 128 registers (kwin_minb) the one-tile warps win below 500 tiles
    // when the chain of depth passes is short (M <= 600; profiles/r02/kwin_nct1_minb4_r02.jsonl,
    // kwin_nct1_threshold_r02.jsonl): 1000 columns 26.0, 2000 27.7, 2500 27.7, 3334 28.4 against
    // 28.0 for (1,4,2,2); even at 4000; behind from 5000 (28.7 vs 29.0).  The n = 60000 shard
    // (938 depths, 3750 columns) keeps two-tile warps: 28.7 against 26.5.
    if (b8 == 8 && (ntile >= 500 || M > 600)) { D = 1; CW = 4; NCT = 2; K = 2; }
    else if (b8 == 8) { D = 1; CW = 4; NCT = 1; K = 2; }
    else if (b8 == 4 && ntile < 2000) { D = 4; CW = 2; NCT = 2; }
    else { D = 2; CW = 2; NCT = 2; }   // also the default of the small menu (nbw != 8/16/32/64)
}

int make_plan(int64_t n, int64_t nbw, int64_t nev, const elpa_b200_opts *o, Plan &p) {
    int kernel = o ? o->kernel : ELPA_B200_KERNEL_AUTO;
    if (kernel < ELPA_B200_KERNEL_AUTO || kernel > ELPA_B200_KERNEL_DFMA) return ELPA_B200_ERR_ARG;
    if (kernel == ELPA_B200_KERNEL_AUTO)
        kernel = b8_supported(nbw) ? ELPA_B200_KERNEL_DMMA : ELPA_B200_KERNEL_REFERENCE;
    if (kernel == ELPA_B200_KERNEL_DMMA && !b8_supported(nbw)) return ELPA_B200_ERR_ARG;
    p.kernel = kernel;
    p.nbw = nbw;
    if (kernel == ELPA_B200_KERNEL_REFERENCE) {
        p.threads = 128;
        p.grid = (nev + 127) / 128;
        p.ws_bytes = 0;
        return ELPA_B200_OK;
    }
    const int64_t M = num_depths(n, nbw);
    if (kernel == ELPA_B200_KERNEL_DFMA) {
        // lane-per-column FP64 CUDA-core kernel: k reflectors fused per group (fused_k, default
        // 8: measured best of 2/4/6/8), CW = 2 warps per CTA
        const int kf = (o && o->fused_k) ? o->fused_k : 8;
        const int CW = (o && o->col_warps) ? o->col_warps : 2;
        if ((o && (o->depth_warps > 1 || o->tiles_per_warp > 1 || o->groups_per_step > 1)) || !dfma_compiled(nbw, kf, CW))
            return ELPA_B200_ERR_ARG;
        p.kf = kf; p.CW = CW; p.D = 1; p.NCT = 1; p.K = 1;
        p.grid_req = o ? o->grid_ctas : 0;
        if (p.grid_req < 0) return ELPA_B200_ERR_ARG;
        p.nx = (nev + 16 * CW - 1) / (16 * CW);           // two lanes per column: 16 columns per warp
        p.items = p.nx * M;
        p.grid = p.items;
        p.threads = 32 * CW;
        p.smem = size_t(4) * dfma_blob_doubles(int(nbw), kf) * 8 + 2 * 4 * 8 + 16;   // DfmaCfg::SMEM
        const int64_t blobs = (M > 0) ? dfma_total_groups(n, nbw, kf) * dfma_blob_doubles(int(nbw), kf) * 8 : 0;
        p.gb_off = (blobs + 255) / 256 * 256;
        p.ws_bytes = (M > 0) ? p.gb_off + (M + 1) * 8 : 0;
        return ELPA_B200_OK;
    }
    if (o && o->fused_k) return ELPA_B200_ERR_ARG;           // fused_k is a DFMA-kernel knob
    p.b8 = int(nbw / 8);
    const int64_t ntile = (nev + 7) / 8;
    int D = o ? o->depth_warps : 0, CW = o ? o->col_warps : 0, NCT = o ? o->tiles_per_warp : 0;
    int K = o ? o->groups_per_step : 0;
    if (D == 0 && CW == 0 && NCT == 0) {
        int Ka = 0;
        auto_shape(ntile, M, p.b8, D, CW, NCT, Ka);
        if (K == 0) K = Ka;
    }
    if (K == 0) K = 1;
    const bool kwin = K >= 2 && kwin_compiled(p.b8, D, CW, NCT, K);
    if (!kwin && !shape_compiled(D, CW, NCT, K, p.b8)) return ELPA_B200_ERR_ARG;
    p.D = D; p.CW = CW; p.NCT = NCT; p.K = K;
    p.grid_req = o ? o->grid_ctas : 0;
    if (p.grid_req < 0) return ELPA_B200_ERR_ARG;
    p.nx = (ntile + CW * NCT - 1) / (CW * NCT);
    p.items = p.nx * ((M + D - 1) / D);
    p.grid = p.items;          // capped by co-residency at launch
    p.threads = 32 * D * CW;
    p.smem = kwin ? kwin_smem(p.b8, CW, NCT, K, kwin_stages(p.b8, CW, NCT, K)) : dmma_smem(p.b8, D, CW, NCT, K);
    if (p.smem > size_t(smem_optin())) return ELPA_B200_ERR_ARG;   // shape does not fit this nbw
    p.ws_bytes = (M > 0) ? total_groups(n, p.b8, M) * blob_doubles(p.b8 + 1, 0) * 8 : 0;
    return ELPA_B200_OK;
}

int validate(int64_t n, int64_t nbw, int64_t nev, const void *hh_v, const void *hh_tau, const void *Q,
             int64_t ldq, bool check_q_align) {
    if (n < 0 || nbw < 1 || nev < 0 || nev > n || ldq < (n > 1 ? n : 1) || n > kMaxN) return ELPA_B200_ERR_ARG;
    const int64_t R = hh_total(n, nbw);
    if (R > 0 && nev > 0 && (!hh_v || !hh_tau || !Q)) return ELPA_B200_ERR_NULL;
    if (check_q_align && R > 0 && nev > 0 && ((ldq & 1) || (reinterpret_cast<uintptr_t>(Q) & 15)))
        return ELPA_B200_ERR_ALIGN;
    return ELPA_B200_OK;
}

// groups [g_lo, g_hi) of every depth (g_hi < 0: all groups)
template <int B8>
int launch_prep(int64_t n, const double *hh_v, const double *hh_tau, double *ws, cudaStream_t s, int64_t g_lo = 0,
                int64_t g_hi = -1) {
    const int64_t M = num_depths(n, 8 * B8);
    const int64_t G0 = groups_at_depth(n, B8, 0);
    if (g_hi < 0 || g_hi > G0) g_hi = G0;
    if (g_lo >= g_hi || M == 0) return ELPA_B200_OK;
    dim3 grid(unsigned((g_hi - g_lo + 3) / 4), unsigned(M));
    prep_dmma_kernel<B8, 0><<<grid, 128, 0, s>>>(n, hh_v, hh_tau, ws, g_lo, g_hi);
    return cudaGetLastError() == cudaSuccess ? ELPA_B200_OK : ELPA_B200_ERR_CUDA;
}

template <int B, int KF>
int launch_prep_dfma(const Plan &p, int64_t n, const double *hh_v, const double *hh_tau, char *ws, cudaStream_t s,
                     int64_t g_lo = 0, int64_t g_hi = -1) {
    const int64_t M = num_depths(n, B);
    const int64_t G0 = dfma_groups(n, B, KF, 0);
    if (g_hi < 0 || g_hi > G0) g_hi = G0;
    int64_t *gbase = reinterpret_cast<int64_t *>(ws + p.gb_off);
    if (g_lo == 0) dfma_gbase_kernel<<<1, 1, 0, s>>>(n, B, KF, M, gbase);
    if (g_lo >= g_hi || M == 0) return cudaGetLastError() == cudaSuccess ? ELPA_B200_OK : ELPA_B200_ERR_CUDA;
    dim3 grid(unsigned(std::min<int64_t>(64, ((g_hi - g_lo) * dfma_blob_doubles(B, KF) + 255) / 256)), unsigned(M));
    prep_dfma_kernel<B, KF><<<grid, 256, 0, s>>>(n, hh_v, hh_tau, gbase, reinterpret_cast<double *>(ws), g_lo, g_hi);
    return cudaGetLastError() == cudaSuccess ? ELPA_B200_OK : ELPA_B200_ERR_CUDA;
}

template <int B, int KF, int CW>
int launch_dfma(const Plan &p, int64_t n, int64_t nev, const char *ws, double *Q, int64_t ldq, cudaStream_t s) {
    auto kern = apply_dfma_kernel<B, KF, CW>;
    const size_t smem = DfmaCfg<B, KF, CW>::SMEM;
    int per_sm = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, DfmaCfg<B, KF, CW>::THREADS, smem) != cudaSuccess ||
        per_sm < 1)
        return fail_cuda();
    int64_t grid = int64_t(per_sm) * sm_count();
    if (p.grid_req > 0 && p.grid_req < grid) grid = p.grid_req;
    if (grid > p.items) grid = p.items;
    uint64_t *prog = nullptr;
    const size_t pbytes = size_t(p.items * CW + 1) * 8;   // one word per (item, column warp) + counter
    if (lib_malloc_async(reinterpret_cast<void **>(&prog), pbytes, s) != cudaSuccess) return fail_cuda();
    int rc = cudaMemsetAsync(prog, 0, pbytes, s) == cudaSuccess ? ELPA_B200_OK : ELPA_B200_ERR_CUDA;
    if (rc == ELPA_B200_OK) {
        kern<<<unsigned(grid), DfmaCfg<B, KF, CW>::THREADS, smem, s>>>(
            n, nev, reinterpret_cast<const double *>(ws), reinterpret_cast<const int64_t *>(ws + p.gb_off), Q, ldq,
            prog, pub_period());
        if (cudaGetLastError() != cudaSuccess) rc = ELPA_B200_ERR_CUDA;
    }
    if (cudaFreeAsync(prog, s) != cudaSuccess && rc == ELPA_B200_OK) rc = ELPA_B200_ERR_CUDA;
    return rc;
}

// dispatch over the compiled (nbw, k) menu of the DFMA kernel (CW = 2)
template <class F>
int dfma_dispatch(int64_t nbw, int kf, F &&f) {
#define ELPA_DFMA_K(B_)                                                          \
    if (nbw == B_) {                                                             \
        if (kf == 2) return f(std::integral_constant<int, B_>{}, std::integral_constant<int, 2>{}); \
        if (kf == 4) return f(std::integral_constant<int, B_>{}, std::integral_constant<int, 4>{}); \
        if (kf == 6) return f(std::integral_constant<int, B_>{}, std::integral_constant<int, 6>{}); \
        if (kf == 8) return f(std::integral_constant<int, B_>{}, std::integral_constant<int, 8>{}); \
    }
    ELPA_DFMA_K(8) ELPA_DFMA_K(16) ELPA_DFMA_K(32) ELPA_DFMA_K(64)
#undef ELPA_DFMA_K
    return ELPA_B200_ERR_ARG;
}

// Grid of the persistent item kernel: the co-resident maximum (more CTAs could not run
// concurrently anyway; correctness does not depend on co-residency, see kernel_dmma.cuh).
template <int KIND, int B8, int D, int CW, int NCT, int K>
int64_t dmma_grid(const Plan &p) {
    auto kern = apply_dmma_kernel<KIND, B8, D, CW, NCT, K>;
    const size_t smem = DmmaCfg<KIND, B8, D, CW, NCT, K>::SMEM;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, DmmaCfg<KIND, B8, D, CW, NCT, K>::THREADS, smem) !=
            cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        return -1;
    }
    int64_t g = int64_t(per_sm) * sm_count();
    if (p.grid_req > 0 && p.grid_req < g) g = p.grid_req;
    return g < p.items ? g : p.items;
}

template <int KIND, int B8, int D, int CW, int NCT, int K>
int launch_dmma_shape(const Plan &p, int64_t n, int64_t nev, const double *ws, double *Q, int64_t ldq,
                      cudaStream_t s) {
    const int64_t grid = dmma_grid<KIND, B8, D, CW, NCT, K>(p);
    if (grid < 1) return ELPA_B200_ERR_CUDA;
    uint64_t *prog = nullptr;
    // one progress word per work item + the work-item counter, zeroed per launch
    const size_t pbytes = size_t(p.items + 1) * 8;
    if (lib_malloc_async(reinterpret_cast<void **>(&prog), pbytes, s) != cudaSuccess) return fail_cuda();
    int rc = ELPA_B200_OK;
    if (cudaMemsetAsync(prog, 0, pbytes, s) != cudaSuccess) rc = ELPA_B200_ERR_CUDA;
    if (rc == ELPA_B200_OK) {
        apply_dmma_kernel<KIND, B8, D, CW, NCT, K><<<unsigned(grid), DmmaCfg<KIND, B8, D, CW, NCT, K>::THREADS,
                                                     DmmaCfg<KIND, B8, D, CW, NCT, K>::SMEM, s>>>(n, nev, ws, Q, ldq, prog,
                                                                                                  pub_period((nev + 7) / 8));
        if (cudaGetLastError() != cudaSuccess) rc = ELPA_B200_ERR_CUDA;
    }
    if (cudaFreeAsync(prog, s) != cudaSuccess && rc == ELPA_B200_OK) rc = ELPA_B200_ERR_CUDA;
    return rc;
}

template <int B8, int CW, int NCT, int K>
int launch_kwin_shape(const Plan &p, int64_t n, int64_t nev, const double *ws, double *Q, int64_t ldq, cudaStream_t s) {
    using Cfg = KwinCfg<B8, CW, NCT, K>;
    auto kern = apply_dmma_kwin_kernel<B8, CW, NCT, K>;
    int per_sm = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM)) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::THREADS, Cfg::SMEM) != cudaSuccess ||
        per_sm < 1)
        return fail_cuda();
    int64_t grid = int64_t(per_sm) * sm_count();
    if (p.grid_req > 0 && p.grid_req < grid) grid = p.grid_req;
    if (grid > p.items) grid = p.items;
    uint64_t *prog = nullptr;
    const size_t pbytes = size_t(p.items * CW + 1) * 8;   // one word per (item, column warp) + counter
    if (lib_malloc_async(reinterpret_cast<void **>(&prog), pbytes, s) != cudaSuccess) return fail_cuda();
    int rc = cudaMemsetAsync(prog, 0, pbytes, s) == cudaSuccess ? ELPA_B200_OK : ELPA_B200_ERR_CUDA;
    if (rc == ELPA_B200_OK) {
        kern<<<unsigned(grid), Cfg::THREADS, Cfg::SMEM, s>>>(n, nev, ws, Q, ldq, prog, kwin_pub_period((nev + 7) / 8));
        if (cudaGetLastError() != cudaSuccess) rc = ELPA_B200_ERR_CUDA;
    }
    if (cudaFreeAsync(prog, s) != cudaSuccess && rc == ELPA_B200_OK) rc = ELPA_B200_ERR_CUDA;
    return rc;
}

template <int B8>
int launch_dmma_b8(const Plan &p, int64_t n, int64_t nev, const double *ws, double *Q, int64_t ldq,
                   cudaStream_t s) {
    if constexpr (B8 == 4 || B8 == 8) {
#define ELPA_KWIN(D_, CW_, NCT_, K_)                            \
        if (p.D == D_ && p.CW == CW_ && p.NCT == NCT_ && p.K == K_) \
            return launch_kwin_shape<B8, CW_, NCT_, K_>(p, n, nev, ws, Q, ldq, s);
        if (p.K >= 2) {
            ELPA_KWIN_SHAPES(ELPA_KWIN)
        }
#undef ELPA_KWIN
    }
#define ELPA_SHAPE(D_, CW_, NCT_, K_)                          \
    if (p.D == D_ && p.CW == CW_ && p.NCT == NCT_ && p.K == K_) \
        return launch_dmma_shape<KIND_DMMA, B8, D_, CW_, NCT_, K_>(p, n, nev, ws, Q, ldq, s);
    if constexpr (B8 == 1 || B8 == 2 || B8 == 4 || B8 == 8) {
        ELPA_SHAPES(ELPA_SHAPE)
    } else {
        ELPA_SMALL_SHAPES(ELPA_SHAPE)
    }
#undef ELPA_SHAPE
    return ELPA_B200_ERR_ARG;
}

// Groups whose every sweep is < sweep (all groups when sweep >= n - 2): group g holds the sweeps
// k*g - 1 .. k*g + k - 2 (k = 8 for DMMA, fused_k for DFMA)
int64_t groups_complete(const Plan &p, int64_t n, int64_t sweep) {
    const int64_t k = p.kernel == ELPA_B200_KERNEL_DFMA ? p.kf : 8;
    const int64_t G0 = p.kernel == ELPA_B200_KERNEL_DFMA ? dfma_groups(n, p.nbw, k, 0) : groups_at_depth(n, p.b8, 0);
    if (sweep >= n - 2) return G0;
    if (sweep < k - 1) return 0;
    return std::min<int64_t>(G0, (sweep - k + 1) / k + 1);
}

// prepare the groups complete for sweeps < sweep_hi that were not complete for sweeps < sweep_lo
int prepare_impl(const Plan &p, int64_t n, const double *hh_v, const double *hh_tau, void *ws, cudaStream_t s,
                 int64_t sweep_lo = 0, int64_t sweep_hi = INT64_MAX) {
    if (p.kernel == ELPA_B200_KERNEL_REFERENCE || p.ws_bytes == 0) return ELPA_B200_OK;
    const int64_t g_lo = sweep_lo <= 0 ? 0 : groups_complete(p, n, sweep_lo);
    const int64_t g_hi = groups_complete(p, n, sweep_hi);
    if (p.kernel == ELPA_B200_KERNEL_DFMA)
        return dfma_dispatch(p.nbw, p.kf, [&](auto b, auto k) {
            return launch_prep_dfma<decltype(b)::value, decltype(k)::value>(p, n, hh_v, hh_tau, static_cast<char *>(ws), s,
                                                                          g_lo, g_hi);
        });
    double *w = static_cast<double *>(ws);
    switch (p.b8) {
#define ELPA_PREP_CASE(B8_) \
    case B8_: return launch_prep<B8_>(n, hh_v, hh_tau, w, s, g_lo, g_hi);
        ELPA_PREP_CASE(1) ELPA_PREP_CASE(2) ELPA_PREP_CASE(3) ELPA_PREP_CASE(4) ELPA_PREP_CASE(5) ELPA_PREP_CASE(6)
        ELPA_PREP_CASE(7) ELPA_PREP_CASE(8) ELPA_PREP_CASE(9) ELPA_PREP_CASE(10) ELPA_PREP_CASE(11)
        ELPA_PREP_CASE(12) ELPA_PREP_CASE(13) ELPA_PREP_CASE(14) ELPA_PREP_CASE(15) ELPA_PREP_CASE(16)
#undef ELPA_PREP_CASE
    }
    return ELPA_B200_ERR_ARG;
}

int apply_impl(const Plan &p, int64_t n, int64_t nbw, int64_t nev, const double *hh_v, const double *hh_tau,
               const void *ws, double *Q, int64_t ldq, cudaStream_t s) {
    if (p.kernel == ELPA_B200_KERNEL_REFERENCE) {
        apply_reference_kernel<<<unsigned(p.grid), p.threads, 0, s>>>(n, nbw, nev, hh_v, hh_tau, Q, ldq);
        return cudaGetLastError() == cudaSuccess ? ELPA_B200_OK : ELPA_B200_ERR_CUDA;
    }
    if (p.kernel == ELPA_B200_KERNEL_DFMA)
        return dfma_dispatch(p.nbw, p.kf, [&](auto b, auto k) {
            return launch_dfma<decltype(b)::value, decltype(k)::value, 2>(p, n, nev, static_cast<const char *>(ws), Q,
                                                                         ldq, s);
        });
    const double *w = static_cast<const double *>(ws);
    switch (p.b8) {
#define ELPA_APPLY_CASE(B8_) \
    case B8_: return launch_dmma_b8<B8_>(p, n, nev, w, Q, ldq, s);
        ELPA_APPLY_CASE(1) ELPA_APPLY_CASE(2) ELPA_APPLY_CASE(3) ELPA_APPLY_CASE(4) ELPA_APPLY_CASE(5)
        ELPA_APPLY_CASE(6) ELPA_APPLY_CASE(7) ELPA_APPLY_CASE(8) ELPA_APPLY_CASE(9) ELPA_APPLY_CASE(10)
        ELPA_APPLY_CASE(11) ELPA_APPLY_CASE(12) ELPA_APPLY_CASE(13) ELPA_APPLY_CASE(14) ELPA_APPLY_CASE(15)
        ELPA_APPLY_CASE(16)
#undef ELPA_APPLY_CASE
    }
    return ELPA_B200_ERR_ARG;
}

// Host-side record of prepared workspaces: apply_prepared must read the layout
// prepare wrote, and a DMMA-prepared workspace also passes the DFMA size check.  prepare records
// (pointer, kernel, b8, n) here; apply_prepared returns ERR_ARG when the pointer was prepared for
// a different kernel, nbw or n.  Pointers the table has not seen (prepared by another process,
// or evicted after 256 newer preparations) are not checked.
struct PreparedTag { const void *ws = nullptr; int kernel = 0, b8 = 0; int64_t n = 0; };
std::mutex g_tag_mu;
PreparedTag g_tags[256];
int g_tag_next = 0;

void record_prepared(const void *ws, const Plan &p, int64_t n) {
    std::lock_guard<std::mutex> lock(g_tag_mu);
    for (PreparedTag &t : g_tags)
        if (t.ws == ws) { t.kernel = p.kernel; t.b8 = p.b8; t.n = n; return; }
    g_tags[g_tag_next] = PreparedTag{ws, p.kernel, p.b8, n};
    g_tag_next = (g_tag_next + 1) % 256;
}

bool prepared_matches(const void *ws, const Plan &p, int64_t n) {
    std::lock_guard<std::mutex> lock(g_tag_mu);
    for (const PreparedTag &t : g_tags)
        if (t.ws == ws) return t.kernel == p.kernel && t.b8 == p.b8 && t.n == n;
    return true;
}

}  // namespace

extern "C" {

int elpa_b200_set_workspace_cache(int enable) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail_cuda();
    return set_pool_caching(dev, enable != 0) ? ELPA_B200_OK : fail_cuda();
}

int elpa_b200_release_cache(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail_cuda();
    cudaMemPool_t pool = lib_pool(dev);
    if (pool && cudaMemPoolTrimTo(pool, 0) != cudaSuccess) return fail_cuda();
    return ELPA_B200_OK;
}

int64_t elpa_hh_count(int64_t n, int64_t nbw) {
    if (n < 0 || nbw < 1) return -1;
    return hh_total(n, nbw);
}

int64_t elpa_hh_offset(int64_t n, int64_t nbw, int64_t j) {
    if (n < 0 || nbw < 1 || j < 0) return -1;
    const int64_t R = hh_total(n, nbw);
    if (R == 0) return 0;
    if (j >= n - 2) return R;
    return hh_off(j, n, nbw);
}

const char *elpa_b200_strerror(int code) {
    switch (code) {
        case ELPA_B200_OK: return "ok";
        case ELPA_B200_ERR_ARG: return "invalid argument (n, nbw, nev, ldq or options)";
        case ELPA_B200_ERR_NULL: return "required pointer is NULL";
        case ELPA_B200_ERR_ALIGN: return "misaligned Q (FP64: ldq even; FP32: ldq % 4 == 0; Q 16-byte aligned) or workspace";
        case ELPA_B200_ERR_DEVICE: return "current device is not an sm_100 (B200) GPU";
        case ELPA_B200_ERR_CUDA: return "CUDA runtime error or kernel launch failure";
        case ELPA_B200_ERR_SPACE: return "workspace too small";
    }
    return "unknown error code";
}

int64_t elpa_b200_workspace_bytes(int64_t n, int64_t nbw, const elpa_b200_opts *opts) {
    if (n < 0 || nbw < 1) return -1;
    Plan p;
    if (make_plan(n, nbw, n > 0 ? n : 1, opts, p) != ELPA_B200_OK) return -1;
    return p.ws_bytes;
}

int elpa_b200_describe(int64_t n, int64_t nbw, int64_t nev, const elpa_b200_opts *opts, char *buf, size_t buflen) {
    if (n < 0 || nbw < 1 || nev < 0 || nev > n) return ELPA_B200_ERR_ARG;
    Plan p;
    int rc = make_plan(n, nbw, nev, opts, p);
    if (rc != ELPA_B200_OK) return rc;
    if (buf && buflen)
        snprintf(buf, buflen,
                 "kernel=%s b8=%d D=%d CW=%d NCT=%d K=%d k=%d items=%lld grid_req=%d block=%d smem=%zu ws=%lld",
                 p.kernel == ELPA_B200_KERNEL_DMMA ? "dmma" : (p.kernel == ELPA_B200_KERNEL_DFMA ? "dfma" : "reference"),
                 p.b8, p.D, p.CW, p.NCT, p.K, p.kernel == ELPA_B200_KERNEL_DFMA ? p.kf : 8, (long long)p.items,
                 p.grid_req, p.threads, p.smem, (long long)p.ws_bytes);
    if (hh_total(n, nbw) == 0 || nev == 0) return 0;
    return p.kernel == ELPA_B200_KERNEL_REFERENCE ? 1 : 2;
}

int elpa_b200_prepare(int64_t n, int64_t nbw, const double *hh_v, const double *hh_tau, void *workspace,
                      size_t workspace_bytes, elpa_b200_stream_t stream, const elpa_b200_opts *opts) {
    if (n < 0 || nbw < 1) return ELPA_B200_ERR_ARG;
    Plan p;
    int rc = make_plan(n, nbw, n > 0 ? n : 1, opts, p);
    if (rc != ELPA_B200_OK) return rc;
    if (hh_total(n, nbw) == 0 || p.ws_bytes == 0) return ELPA_B200_OK;
    if (!hh_v || !hh_tau || !workspace) return ELPA_B200_ERR_NULL;
    if (reinterpret_cast<uintptr_t>(workspace) & 255) return ELPA_B200_ERR_ALIGN;
    if (workspace_bytes < size_t(p.ws_bytes)) return ELPA_B200_ERR_SPACE;
    if ((rc = check_device()) != ELPA_B200_OK) return rc;
    rc = prepare_impl(p, n, hh_v, hh_tau, workspace, reinterpret_cast<cudaStream_t>(stream));
    if (rc == ELPA_B200_OK) record_prepared(workspace, p, n);
    return rc;
}

int elpa_b200_prepare_sweeps(int64_t n, int64_t nbw, const double *hh_v, const double *hh_tau, void *workspace,
                             size_t workspace_bytes, int64_t sweep_lo, int64_t sweep_hi, elpa_b200_stream_t stream,
                             const elpa_b200_opts *opts) {
    if (n < 0 || nbw < 1 || sweep_lo < 0 || sweep_hi < sweep_lo) return ELPA_B200_ERR_ARG;
    Plan p;
    int rc = make_plan(n, nbw, n > 0 ? n : 1, opts, p);
    if (rc != ELPA_B200_OK) return rc;
    if (hh_total(n, nbw) == 0 || p.ws_bytes == 0) return ELPA_B200_OK;
    if (!hh_v || !hh_tau || !workspace) return ELPA_B200_ERR_NULL;
    if (reinterpret_cast<uintptr_t>(workspace) & 255) return ELPA_B200_ERR_ALIGN;
    if (workspace_bytes < size_t(p.ws_bytes)) return ELPA_B200_ERR_SPACE;
    if ((rc = check_device()) != ELPA_B200_OK) return rc;
    rc = prepare_impl(p, n, hh_v, hh_tau, workspace, reinterpret_cast<cudaStream_t>(stream), sweep_lo, sweep_hi);
    if (rc == ELPA_B200_OK && sweep_hi >= n - 2) record_prepared(workspace, p, n);
    return rc;
}

int elpa_b200_apply_prepared(int64_t n, int64_t nbw, int64_t nev, const double *hh_v, const double *hh_tau,
                             const void *workspace, size_t workspace_bytes, double *Q, int64_t ldq,
                             elpa_b200_stream_t stream, const elpa_b200_opts *opts) {
    Plan p;
    int rc = validate(n, nbw, nev, (opts && opts->kernel == ELPA_B200_KERNEL_REFERENCE) ? hh_v : (const void *)1,
                      (opts && opts->kernel == ELPA_B200_KERNEL_REFERENCE) ? hh_tau : (const void *)1, Q, ldq, true);
    if (rc != ELPA_B200_OK) return rc;
    if ((rc = make_plan(n, nbw, nev, opts, p)) != ELPA_B200_OK) return rc;
    if (hh_total(n, nbw) == 0 || nev == 0) return ELPA_B200_OK;
    if (p.kernel == ELPA_B200_KERNEL_REFERENCE && (!hh_v || !hh_tau)) return ELPA_B200_ERR_NULL;
    if (p.kernel != ELPA_B200_KERNEL_REFERENCE) {
        if (!workspace) return ELPA_B200_ERR_NULL;
        if (reinterpret_cast<uintptr_t>(workspace) & 255) return ELPA_B200_ERR_ALIGN;
        if (workspace_bytes < size_t(p.ws_bytes)) return ELPA_B200_ERR_SPACE;
        if (!prepared_matches(workspace, p, n)) return ELPA_B200_ERR_ARG;
    }
    if ((rc = check_device()) != ELPA_B200_OK) return rc;
    return apply_impl(p, n, nbw, nev, hh_v, hh_tau, workspace, Q, ldq, reinterpret_cast<cudaStream_t>(stream));
}

int elpa_trans_ev_tridi_to_band_ex(int64_t n, int64_t nbw, int64_t nev, const double *hh_v, const double *hh_tau,
                                   double *Q, int64_t ldq, elpa_b200_stream_t stream, const elpa_b200_opts *opts) {
    int rc = validate(n, nbw, nev, hh_v, hh_tau, Q, ldq, true);
    if (rc != ELPA_B200_OK) return rc;
    Plan p;
    if ((rc = make_plan(n, nbw, nev, opts, p)) != ELPA_B200_OK) return rc;
    if (hh_total(n, nbw) == 0 || nev == 0) return ELPA_B200_OK;
    if ((rc = check_device()) != ELPA_B200_OK) return rc;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    void *ws = nullptr;
    if (p.ws_bytes > 0 && lib_malloc_async(&ws, size_t(p.ws_bytes), s) != cudaSuccess) return fail_cuda();
    rc = prepare_impl(p, n, hh_v, hh_tau, ws, s);
    if (rc == ELPA_B200_OK) rc = apply_impl(p, n, nbw, nev, hh_v, hh_tau, ws, Q, ldq, s);
    if (ws && cudaFreeAsync(ws, s) != cudaSuccess && rc == ELPA_B200_OK) rc = ELPA_B200_ERR_CUDA;
    return rc;
}

int elpa_trans_ev_tridi_to_band(int64_t n, int64_t nbw, int64_t nev, const double *hh_v, const double *hh_tau,
                                double *Q, int64_t ldq, elpa_b200_stream_t stream) {
    return elpa_trans_ev_tridi_to_band_ex(n, nbw, nev, hh_v, hh_tau, Q, ldq, stream, nullptr);
}

int elpa_trans_ev_tridi_to_band_host(int64_t n, int64_t nbw, int64_t nev, const double *hh_v, const double *hh_tau,
                                     double *Q, int64_t ldq, elpa_b200_stream_t stream, const elpa_b200_opts *opts) {
    int rc = validate(n, nbw, nev, hh_v, hh_tau, Q, ldq, false);
    if (rc != ELPA_B200_OK) return rc;
    if (ldq & 1) return ELPA_B200_ERR_ALIGN;
    Plan p;
    if ((rc = make_plan(n, nbw, nev, opts, p)) != ELPA_B200_OK) return rc;
    const int64_t R = hh_total(n, nbw);
    if (R == 0 || nev == 0) return ELPA_B200_OK;
    if ((rc = check_device()) != ELPA_B200_OK) return rc;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    using wall = std::chrono::steady_clock;
    const auto w_enter = wall::now();
    auto wall_ms = [&](wall::time_point t) { return std::chrono::duration<double, std::milli>(t - w_enter).count(); };
    wall::time_point w_alloc = w_enter, w_enqueued = w_enter;

    // Column blocks of CH eigenvectors stream through NBUF device buffers: H2D on one copy
    // stream, apply on `stream`, D2H on another, so PCIe traffic overlaps the kernel (columns
    // are independent: each block's result is bitwise the unblocked one).
    // Block schedule [e, m, e], e = nev/10: a thin first block (its upload shares PCIe with the
    // reflectors and delays the first launch; its compute covers the wide block's upload) and a
    // thin last one (its download is the exposed tail; its compute covers the wide block's
    // download), one wide middle block (wide stripes run the kernel faster: 30.4 TF/s at 16000
    // columns, 29.6 at 8000, 28.1 at 3336).  Measured at C3: 6 equal blocks 616 ms, 4 equal 612 ms
    // (profiles/r02/host_blocks_r02.log).  Below 4000 eigenvectors: two equal blocks.
    // Development override ELPA_B200_HOST_BLOCKS = k: k equal blocks.
    static const int64_t kBlocks = [] {
        const char *e = getenv("ELPA_B200_HOST_BLOCKS");
        const int64_t v = e ? atoll(e) : 0;
        return v >= 1 ? v : 0;
    }();
    std::vector<int64_t> bstart;                       // block c = columns [bstart[c], bstart[c+1])
    auto r8 = [](int64_t x) { return std::max<int64_t>(8, (x + 7) / 8 * 8); };
    if (kBlocks == 0 && nev >= 4000) {
        const int64_t e = r8(nev / 10);
        for (int64_t c0 : {int64_t(0), e, nev - e}) bstart.push_back(c0);
    } else {
        const int64_t k = kBlocks ? kBlocks : 2;         // few columns: the reflector upload dominates
        const int64_t ch = r8((nev + k - 1) / k);
        for (int64_t c0 = 0; c0 < nev; c0 += ch) bstart.push_back(c0);
    }
    bstart.push_back(nev);
    bstart.erase(std::unique(bstart.begin(), bstart.end()), bstart.end());
    const int64_t nblk = int64_t(bstart.size()) - 1;
    int64_t CH = 8;
    for (int64_t c = 0; c < nblk; c++) CH = std::max(CH, bstart[c + 1] - bstart[c]);
    constexpr int NBUF = 3;
    const size_t bqc = size_t(ldq) * CH * 8, bv = size_t(R) * nbw * 8, bt = size_t(R) * 8;
    auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
    const size_t off_v = 0, off_t = up(bv), off_w = off_t + up(bt), off_q = off_w + up(size_t(p.ws_bytes));
    const size_t total = off_q + NBUF * up(bqc);
    char *buf = nullptr;
    if (lib_malloc_async(reinterpret_cast<void **>(&buf), total, s) != cudaSuccess) return fail_cuda();
    w_alloc = wall::now();
    double *dv = reinterpret_cast<double *>(buf + off_v), *dt = reinterpret_cast<double *>(buf + off_t);
    void *ws = p.ws_bytes ? buf + off_w : nullptr;
    double *dq[NBUF];
    for (int i = 0; i < NBUF; i++) dq[i] = reinterpret_cast<double *>(buf + off_q + i * up(bqc));

    cudaStream_t hs = nullptr, ds = nullptr, cs2 = nullptr;
    std::vector<cudaEvent_t> ev_h2d(nblk), ev_comp(nblk), ev_d2h(nblk);
    cudaEvent_t ev_ready = nullptr, ev_prep = nullptr;
    // ELPA_B200_TRACE=1: timed events, and one JSON line on stderr with every stage's completion
    // time (ms after the buffer allocation): reflector upload + prep, per block H2D/apply/D2H
    static const bool trace = getenv("ELPA_B200_TRACE") != nullptr;
    const unsigned evflags = trace ? cudaEventDefault : cudaEventDisableTiming;
    bool ok = cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&ds, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&cs2, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&ev_ready, evflags) == cudaSuccess &&
              cudaEventCreateWithFlags(&ev_prep, evflags) == cudaSuccess;
    for (int64_t c = 0; ok && c < nblk; c++)
        ok = cudaEventCreateWithFlags(&ev_h2d[c], evflags) == cudaSuccess &&
             cudaEventCreateWithFlags(&ev_comp[c], evflags) == cudaSuccess &&
             cudaEventCreateWithFlags(&ev_d2h[c], evflags) == cudaSuccess;
    if (!ok) rc = ELPA_B200_ERR_CUDA;
    // the buffer is allocated on `s`: the copy streams start after it
    if (rc == ELPA_B200_OK && (cudaEventRecord(ev_ready, s) != cudaSuccess ||
                               cudaStreamWaitEvent(hs, ev_ready, 0) != cudaSuccess))
        rc = ELPA_B200_ERR_CUDA;
    if (rc == ELPA_B200_OK && (cudaMemcpyAsync(dv, hh_v, bv, cudaMemcpyHostToDevice, s) != cudaSuccess ||
                               cudaMemcpyAsync(dt, hh_tau, bt, cudaMemcpyHostToDevice, s) != cudaSuccess))
        rc = ELPA_B200_ERR_CUDA;
    if (rc == ELPA_B200_OK) rc = prepare_impl(p, n, dv, dt, ws, s);
    if (rc == ELPA_B200_OK && cudaEventRecord(ev_prep, s) != cudaSuccess) rc = ELPA_B200_ERR_CUDA;
    // consecutive blocks alternate between `s` and a second compute stream, so the tail of one
    // persistent launch (its last items, with SMs retiring) overlaps the start of the next
    if (rc == ELPA_B200_OK && (cudaStreamWaitEvent(cs2, ev_prep, 0) != cudaSuccess)) rc = ELPA_B200_ERR_CUDA;
    for (int64_t c = 0; rc == ELPA_B200_OK && c < nblk; c++) {
        const int64_t c0 = bstart[c], nc = bstart[c + 1] - c0;
        double *d = dq[c % NBUF];
        cudaStream_t cs = (c & 1) ? cs2 : s;
        // only the n valid rows of each column cross PCIe, in both directions: a legally sized
        // host buffer ends at element (nev-1)*ldq + n, and the padding rows [n, ldq) are never
        // written (the device buffer keeps the pitch ldq; the kernels never read rows >= n)
        const size_t pitch = size_t(ldq) * 8, width = size_t(n) * 8;
        if ((c >= NBUF && cudaStreamWaitEvent(hs, ev_d2h[c - NBUF], 0) != cudaSuccess) ||
            cudaMemcpy2DAsync(d, pitch, Q + c0 * ldq, pitch, width, size_t(nc), cudaMemcpyHostToDevice, hs) !=
                cudaSuccess ||
            cudaEventRecord(ev_h2d[c], hs) != cudaSuccess || cudaStreamWaitEvent(cs, ev_h2d[c], 0) != cudaSuccess) {
            rc = ELPA_B200_ERR_CUDA;
            break;
        }
        Plan pc;
        if ((rc = make_plan(n, nbw, nc, opts, pc)) != ELPA_B200_OK) break;
        if ((rc = apply_impl(pc, n, nbw, nc, dv, dt, ws, d, ldq, cs)) != ELPA_B200_OK) break;
        if (cudaEventRecord(ev_comp[c], cs) != cudaSuccess || cudaStreamWaitEvent(ds, ev_comp[c], 0) != cudaSuccess ||
            cudaMemcpy2DAsync(Q + c0 * ldq, pitch, d, pitch, width, size_t(nc), cudaMemcpyDeviceToHost, ds) !=
                cudaSuccess ||
            cudaEventRecord(ev_d2h[c], ds) != cudaSuccess) {
            rc = ELPA_B200_ERR_CUDA;
            break;
        }
    }
    w_enqueued = wall::now();
    // everything (including work already queued when an error stopped the loop) completes
    // before the buffers go back to the pool
    if (ds) cudaStreamSynchronize(ds);
    if (hs) cudaStreamSynchronize(hs);
    if (cs2) cudaStreamSynchronize(cs2);
    if (cudaFreeAsync(buf, s) != cudaSuccess && rc == ELPA_B200_OK) rc = ELPA_B200_ERR_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess && rc == ELPA_B200_OK) rc = ELPA_B200_ERR_CUDA;
    if (trace && rc == ELPA_B200_OK) {
        auto since = [&](cudaEvent_t e) {
            float ms = -1.0f;
            cudaEventElapsedTime(&ms, ev_ready, e);
            return ms;
        };
        const double w_done = wall_ms(wall::now());
        std::string line = "{\"elpa_b200_trace\": \"host_entry\", \"wall_alloc_ms\": " +
                           std::to_string(wall_ms(w_alloc)) + ", \"wall_enqueued_ms\": " +
                           std::to_string(wall_ms(w_enqueued)) + ", \"wall_done_ms\": " + std::to_string(w_done) +
                           ", \"blocks\": " + std::to_string(nblk) +
                           ", \"cols_per_block\": " + std::to_string(CH) + ", \"prep_done_ms\": " +
                           std::to_string(since(ev_prep)) + ", \"h2d_ms\": [";
        for (int64_t c = 0; c < nblk; c++) line += (c ? ", " : "") + std::to_string(since(ev_h2d[c]));
        line += "], \"apply_ms\": [";
        for (int64_t c = 0; c < nblk; c++) line += (c ? ", " : "") + std::to_string(since(ev_comp[c]));
        line += "], \"d2h_ms\": [";
        for (int64_t c = 0; c < nblk; c++) line += (c ? ", " : "") + std::to_string(since(ev_d2h[c]));
        line += "]}\n";
        fputs(line.c_str(), stderr);
        cudaGetLastError();
    }
    for (int64_t c = 0; c < nblk; c++) {
        if (ev_h2d[c]) cudaEventDestroy(ev_h2d[c]);
        if (ev_comp[c]) cudaEventDestroy(ev_comp[c]);
        if (ev_d2h[c]) cudaEventDestroy(ev_d2h[c]);
    }
    if (ev_ready) cudaEventDestroy(ev_ready);
    if (ev_prep) cudaEventDestroy(ev_prep);
    if (hs) cudaStreamDestroy(hs);
    if (ds) cudaStreamDestroy(ds);
    if (cs2) cudaStreamDestroy(cs2);
    if (rc != ELPA_B200_OK) cudaGetLastError();
    return rc;
}


}  // extern "C"

// ------------------------------------------------------------------------------------------
// Autotuning (header: elpa_b200_autotune_*).  Host-side state machine over candidate options.
// ------------------------------------------------------------------------------------------
struct elpa_b200_autotune {
    int64_t n = 0, nbw = 0, nev = 0;
    int level = 0;
    int dtype = ELPA_B200_DTYPE_F64;
    std::vector<elpa_b200_opts> cand;
    std::vector<double> ms;       // reported time per candidate (< 0: not yet)
    int next = 0;                 // index the next _step returns
    int last = -1;                // index the last _step returned (awaiting _report)
};

namespace {
std::vector<elpa_b200_opts> autotune_candidates_variant(int64_t n, int64_t nbw, int64_t nev, int level, int dtype) {
    // FP32 / complex: FAST = the variant's fast kernel (automatic shape) and, for small problems,
    // its reference kernel; MEDIUM adds every compiled shape of the variant's menu
    std::vector<elpa_b200_opts> c;
    const int fast = dtype == ELPA_B200_DTYPE_F32 ? ELPA_B200_KERNEL_FFMA2 : ELPA_B200_KERNEL_DMMA;
    const bool ok = nbw % 8 == 0 && nbw >= 8 && nbw <= 128;
    elpa_b200_opts o{};
    if (ok) {
        o.kernel = fast;
        c.push_back(o);
    }
    if (!ok || double(hh_total(n, nbw)) * double(nev) * double(nbw) < 2e9) {
        o = elpa_b200_opts{};
        o.kernel = ELPA_B200_KERNEL_REFERENCE;
        c.push_back(o);
    }
    if (level >= ELPA_B200_AUTOTUNE_MEDIUM && ok) {
        int menu[64][4];
        const int cnt = dtype == ELPA_B200_DTYPE_F32 ? f32_shape_menu(int(nbw / 8), menu, 64)
                                                     : c64_shape_menu(int(nbw / 8), menu, 64);
        char buf[8];
        for (int i = 0; i < cnt; i++) {
            o = elpa_b200_opts{};
            o.kernel = fast;
            o.depth_warps = menu[i][0]; o.col_warps = menu[i][1]; o.tiles_per_warp = menu[i][2];
            o.groups_per_step = menu[i][3];
            const int r = dtype == ELPA_B200_DTYPE_F32 ? elpa_b200_describe_f32(n, nbw, nev, &o, buf, sizeof buf)
                                                       : elpa_b200_describe_c64(n, nbw, nev, &o, buf, sizeof buf);
            if (r >= 0) c.push_back(o);
        }
    }
    return c;
}

std::vector<elpa_b200_opts> autotune_candidates(int64_t n, int64_t nbw, int64_t nev, int level) {
    std::vector<elpa_b200_opts> c;
    auto mk = [](int kernel, int D, int CW, int NCT) {
        elpa_b200_opts o{};
        o.kernel = kernel; o.depth_warps = D; o.col_warps = CW; o.tiles_per_warp = NCT;
        o.groups_per_step = (D || CW || NCT) ? 1 : 0;
        return o;
    };
    const bool dmma = b8_supported(nbw);
    const bool dfma = dfma_compiled(nbw, 8, 2);
    if (dmma) c.push_back(mk(ELPA_B200_KERNEL_DMMA, 0, 0, 0));
    if (dfma) c.push_back(mk(ELPA_B200_KERNEL_DFMA, 0, 0, 0));
    // the bit-exact reference kernel is a candidate only where it can finish quickly
    if (!dmma || double(hh_total(n, nbw)) * double(nev) * double(nbw) < 2e9)
        c.push_back(mk(ELPA_B200_KERNEL_REFERENCE, 0, 0, 0));
    if (level >= ELPA_B200_AUTOTUNE_MEDIUM && dmma) {
        const int b8 = int(nbw / 8);
        auto add = [&](const Shape *sh, size_t cnt, int kernel) {
            for (size_t i = 0; i < cnt; i++) {
                elpa_b200_opts o = mk(kernel, sh[i].D, sh[i].CW, sh[i].NCT);
                Plan p;
                if (make_plan(n, nbw, nev, &o, p) == ELPA_B200_OK) c.push_back(o);
            }
        };
        if (b8_full_menu(b8)) {
            add(kShapes, sizeof(kShapes) / sizeof(kShapes[0]), ELPA_B200_KERNEL_DMMA);
            for (const Shape &sh : kKwinShapes) {          // the K-group register-window kernel
                elpa_b200_opts o = mk(ELPA_B200_KERNEL_DMMA, sh.D, sh.CW, sh.NCT);
                o.groups_per_step = sh.K;
                Plan p;
                if (make_plan(n, nbw, nev, &o, p) == ELPA_B200_OK) c.push_back(o);
            }
            for (int kf : {2, 4, 6}) {                  // the DFMA kernel's fused-reflector count
                elpa_b200_opts o = mk(ELPA_B200_KERNEL_DFMA, 0, 0, 0);
                o.fused_k = kf;
                if (dfma) c.push_back(o);
            }
        } else {
            add(kSmallShapes, sizeof(kSmallShapes) / sizeof(kSmallShapes[0]), ELPA_B200_KERNEL_DMMA);
        }
    }
    return c;
}
}  // namespace

extern "C" {

elpa_b200_autotune *elpa_b200_autotune_setup_dtype(int64_t n, int64_t nbw, int64_t nev, int level, int dtype,
                                                  int *error) {
    if (error) *error = ELPA_B200_OK;
    if (n < 0 || nbw < 1 || nev < 0 || nev > n ||
        (level != ELPA_B200_AUTOTUNE_FAST && level != ELPA_B200_AUTOTUNE_MEDIUM) ||
        (dtype != ELPA_B200_DTYPE_F64 && dtype != ELPA_B200_DTYPE_F32 && dtype != ELPA_B200_DTYPE_C64)) {
        if (error) *error = ELPA_B200_ERR_ARG;
        return nullptr;
    }
    auto *at = new elpa_b200_autotune;
    at->n = n; at->nbw = nbw; at->nev = nev; at->level = level; at->dtype = dtype;
    at->cand = dtype == ELPA_B200_DTYPE_F64 ? autotune_candidates(n, nbw, nev, level)
                                            : autotune_candidates_variant(n, nbw, nev, level, dtype);
    at->ms.assign(at->cand.size(), -1.0);
    return at;
}

elpa_b200_autotune *elpa_b200_autotune_setup(int64_t n, int64_t nbw, int64_t nev, int level, int *error) {
    return elpa_b200_autotune_setup_dtype(n, nbw, nev, level, ELPA_B200_DTYPE_F64, error);
}

int elpa_b200_autotune_step(elpa_b200_autotune *at, elpa_b200_opts *opts) {
    if (!at || !opts) return ELPA_B200_ERR_NULL;
    if (at->next >= int(at->cand.size())) return 0;
    at->last = at->next++;
    *opts = at->cand[at->last];
    return 1;
}

int elpa_b200_autotune_report(elpa_b200_autotune *at, double ms) {
    if (!at) return ELPA_B200_ERR_NULL;
    if (at->last < 0 || !(ms > 0.0)) return ELPA_B200_ERR_ARG;
    at->ms[at->last] = ms;
    at->last = -1;
    return ELPA_B200_OK;
}

int elpa_b200_autotune_best(const elpa_b200_autotune *at, elpa_b200_opts *opts, double *ms) {
    if (!at) return ELPA_B200_ERR_NULL;
    int b = -1;
    for (size_t i = 0; i < at->ms.size(); i++)
        if (at->ms[i] > 0.0 && (b < 0 || at->ms[i] < at->ms[b])) b = int(i);
    if (b < 0) return ELPA_B200_ERR_ARG;
    if (opts) *opts = at->cand[b];
    if (ms) *ms = at->ms[b];
    return ELPA_B200_OK;
}

int elpa_b200_autotune_progress(const elpa_b200_autotune *at, int *tried, int *total) {
    if (!at) return ELPA_B200_ERR_NULL;
    int t = 0;
    for (double v : at->ms) t += v > 0.0;
    if (tried) *tried = t;
    if (total) *total = int(at->cand.size());
    return ELPA_B200_OK;
}

int64_t elpa_b200_autotune_save(const elpa_b200_autotune *at, char *buf, size_t buflen) {
    if (!at) return ELPA_B200_ERR_NULL;
    std::string st = "elpa_b200_autotune v2 " + std::to_string(at->n) + " " + std::to_string(at->nbw) + " " +
                     std::to_string(at->nev) + " " + std::to_string(at->level) + " " + std::to_string(at->dtype) +
                     " " + std::to_string(at->next) + " " + std::to_string(at->cand.size());
    char tmp[64];
    for (double v : at->ms) {
        snprintf(tmp, sizeof tmp, " %.17g", v);
        st += tmp;
    }
    const int64_t need = int64_t(st.size()) + 1;
    if (buf && buflen >= size_t(need)) memcpy(buf, st.c_str(), size_t(need));
    return need;
}

elpa_b200_autotune *elpa_b200_autotune_load(const char *state, int *error) {
    if (error) *error = ELPA_B200_ERR_ARG;
    if (!state) {
        if (error) *error = ELPA_B200_ERR_NULL;
        return nullptr;
    }
    long long n, nbw, nev;
    int level, next, cnt, used = 0, dtype = ELPA_B200_DTYPE_F64;
    if (sscanf(state, "elpa_b200_autotune v2 %lld %lld %lld %d %d %d %d%n", &n, &nbw, &nev, &level, &dtype, &next,
               &cnt, &used) != 7 &&
        sscanf(state, "elpa_b200_autotune v1 %lld %lld %lld %d %d %d%n", &n, &nbw, &nev, &level, &next, &cnt,
               &used) != 6)   // v1 snapshots (FP64 only) still load
        return nullptr;
    int err = 0;
    elpa_b200_autotune *at = elpa_b200_autotune_setup_dtype(n, nbw, nev, level, dtype, &err);
    if (!at) return nullptr;
    if (int(at->cand.size()) != cnt || next < 0 || next > cnt) {   // a different build's menu
        delete at;
        return nullptr;
    }
    const char *p = state + used;
    for (int i = 0; i < cnt; i++) {
        int u = 0;
        if (sscanf(p, " %lg%n", &at->ms[i], &u) != 1) {
            delete at;
            return nullptr;
        }
        p += u;
    }
    at->next = next;
    if (error) *error = ELPA_B200_OK;
    return at;
}

void elpa_b200_autotune_destroy(elpa_b200_autotune *at) { delete at; }

int elpa_b200_autotune_run_dtype(int64_t n, int64_t nbw, int64_t nev, int dtype, const void *hh_v, const void *hh_tau,
                                 void *Q_scratch, int64_t ldq, elpa_b200_stream_t stream, int level, int reps,
                                 elpa_b200_opts *best, double *best_ms) {
    if (dtype == ELPA_B200_DTYPE_F64)
        return elpa_b200_autotune_run(n, nbw, nev, static_cast<const double *>(hh_v),
                                      static_cast<const double *>(hh_tau), static_cast<double *>(Q_scratch), ldq,
                                      stream, level, reps, best, best_ms);
    if (!best) return ELPA_B200_ERR_NULL;
    if (reps < 1) reps = 1;
    int err = 0;
    elpa_b200_autotune *at = elpa_b200_autotune_setup_dtype(n, nbw, nev, level, dtype, &err);
    if (!at) return err;
    auto call = [&](const elpa_b200_opts *o) {
        return dtype == ELPA_B200_DTYPE_F32
                   ? elpa_trans_ev_tridi_to_band_f32(n, nbw, nev, static_cast<const float *>(hh_v),
                                                     static_cast<const float *>(hh_tau), static_cast<float *>(Q_scratch),
                                                     ldq, stream, o)
                   : elpa_trans_ev_tridi_to_band_c64(n, nbw, nev, static_cast<const double *>(hh_v),
                                                     static_cast<const double *>(hh_tau),
                                                     static_cast<double *>(Q_scratch), ldq, stream, o);
    };
    int rc = call(nullptr);                          // validation (and a warm-up) through the entry point
    if (rc != ELPA_B200_OK || hh_total(n, nbw) == 0 || nev == 0) {
        if (rc == ELPA_B200_OK) {
            elpa_b200_autotune_step(at, best);
            if (best_ms) *best_ms = 0.0;
        }
        elpa_b200_autotune_destroy(at);
        return rc;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) rc = fail_cuda();
    elpa_b200_opts o;
    while (rc == ELPA_B200_OK && elpa_b200_autotune_step(at, &o) == 1) {
        float bestv = 1e30f;
        for (int r = 0; r < reps && rc == ELPA_B200_OK; r++) {   // whole call: prep + apply
            cudaEventRecord(e0, s);
            rc = call(&o);
            cudaEventRecord(e1, s);
            if (rc == ELPA_B200_OK && cudaEventSynchronize(e1) != cudaSuccess) rc = fail_cuda();
            float ms = 0.f;
            if (rc == ELPA_B200_OK && cudaEventElapsedTime(&ms, e0, e1) == cudaSuccess && ms < bestv) bestv = ms;
        }
        if (rc == ELPA_B200_OK) elpa_b200_autotune_report(at, bestv > 0.f ? bestv : 1e-6);
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (rc == ELPA_B200_OK) rc = elpa_b200_autotune_best(at, best, best_ms);
    elpa_b200_autotune_destroy(at);
    return rc;
}

int elpa_b200_autotune_run(int64_t n, int64_t nbw, int64_t nev, const double *hh_v, const double *hh_tau,
                           double *Q, int64_t ldq, elpa_b200_stream_t stream, int level, int reps,
                           elpa_b200_opts *best, double *best_ms) {
    int rc = validate(n, nbw, nev, hh_v, hh_tau, Q, ldq, true);
    if (rc != ELPA_B200_OK) return rc;
    if (!best) return ELPA_B200_ERR_NULL;
    if (reps < 1) reps = 1;
    int err = 0;
    elpa_b200_autotune *at = elpa_b200_autotune_setup(n, nbw, nev, level, &err);
    if (!at) return err;
    if (hh_total(n, nbw) == 0 || nev == 0) {        // nothing to tune: any option is a no-op
        elpa_b200_autotune_step(at, best);
        if (best_ms) *best_ms = 0.0;
        elpa_b200_autotune_destroy(at);
        return ELPA_B200_OK;
    }
    if ((rc = check_device()) != ELPA_B200_OK) {
        elpa_b200_autotune_destroy(at);
        return rc;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) rc = fail_cuda();
    void *ws[5] = {};                               // prepared reflectors: DMMA, DFMA k = 2/4/6/8
    elpa_b200_opts o;
    while (rc == ELPA_B200_OK && elpa_b200_autotune_step(at, &o) == 1) {
        Plan p;
        if ((rc = make_plan(n, nbw, nev, &o, p)) != ELPA_B200_OK) break;
        const int kind = p.kernel == ELPA_B200_KERNEL_DFMA ? p.kf / 2 : 0;
        if (p.kernel != ELPA_B200_KERNEL_REFERENCE && !ws[kind]) {
            if (lib_malloc_async(&ws[kind], size_t(p.ws_bytes), s) != cudaSuccess) {
                rc = fail_cuda();
                break;
            }
            if ((rc = prepare_impl(p, n, hh_v, hh_tau, ws[kind], s)) != ELPA_B200_OK) break;
        }
        float bestv = 1e30f;
        for (int r = 0; r < reps && rc == ELPA_B200_OK; r++) {
            cudaEventRecord(e0, s);
            rc = apply_impl(p, n, nbw, nev, hh_v, hh_tau, ws[kind], Q, ldq, s);
            cudaEventRecord(e1, s);
            if (rc == ELPA_B200_OK && cudaEventSynchronize(e1) != cudaSuccess) rc = fail_cuda();
            float ms = 0.f;
            if (rc == ELPA_B200_OK && cudaEventElapsedTime(&ms, e0, e1) == cudaSuccess && ms < bestv) bestv = ms;
        }
        if (rc == ELPA_B200_OK) elpa_b200_autotune_report(at, bestv > 0.f ? bestv : 1e-6);
    }
    for (void *w : ws)
        if (w) cudaFreeAsync(w, s);
    cudaStreamSynchronize(s);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (rc == ELPA_B200_OK) rc = elpa_b200_autotune_best(at, best, best_ms);
    elpa_b200_autotune_destroy(at);
    return rc;
}

}  // extern "C"
