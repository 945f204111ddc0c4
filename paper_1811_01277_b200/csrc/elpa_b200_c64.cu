// elpa_b200_c64.cu — C-ABI entry points of the complex Hermitian variant of the hot path (SURVEY
// §8f NEXT-3 second half, include/elpa_b200.h "complex variant"): validation, plan, reflector
// preparation (prep_zmma_kernel) and launch of apply_dmma_kernel<KIND_ZMMA, ...>, or the
// bit-exact reference kernel.  Same geometry and item schedule as the FP64 path.
#include <cuda_runtime.h>

#include <cstdio>

#include "../../include/elpa_b200.h"
#include "geometry.cuh"
#include "host_common.h"
#include "kernel_dmma.cuh"
#include "kernel_dmma_kwin.cuh"
#include "kernel_zprep.cuh"

using namespace elpa_b200;
using namespace elpa_b200_host;

namespace {

// (D depth warps, CW column warps, NZ complex 8-column tiles per warp) menus; the kernel
// template takes NCT = 2*NZ real tiles (Re/Im pairs).  Full menu for nbw = 8/16/32/64.
#define ELPA_Z_SHAPES(X) X(1, 2, 2) X(2, 2, 1) X(1, 2, 1) X(2, 1, 2) X(1, 4, 1) X(2, 2, 2) X(1, 1, 2)
#define ELPA_Z_SMALL_SHAPES(X) X(2, 2, 1) X(1, 2, 1)
struct ZShape { int D, CW, NZ; };
#define ELPA_Z_ENTRY(D_, CW_, NZ_) {D_, CW_, NZ_},
constexpr ZShape kZShapes[] = {ELPA_Z_SHAPES(ELPA_Z_ENTRY)};
constexpr ZShape kZSmallShapes[] = {ELPA_Z_SMALL_SHAPES(ELPA_Z_ENTRY)};

// The K-group register-window kernel (kernel_dmma_kwin.cuh, KIND_ZMMA): D = 1, one complex tile
// per warp, K = 2 groups per step; nbw 32 and 64.
#define ELPA_ZK_SHAPES(X) X(4, 1, 2) X(2, 1, 2) X(8, 1, 2)
struct ZkShape { int CW, NZ, K; };
#define ELPA_ZK_ENTRY(CW_, NZ_, K_) {CW_, NZ_, K_},
constexpr ZkShape kZkShapes[] = {ELPA_ZK_SHAPES(ELPA_ZK_ENTRY)};
bool zk_compiled(int b8, int D, int CW, int NZ, int K) {
    if ((b8 != 4 && b8 != 8) || D != 1) return false;
    for (const ZkShape &s : kZkShapes)
        if (s.CW == CW && s.NZ == NZ && s.K == K) return true;
    return false;
}

bool z_full_menu(int b8) { return b8 == 1 || b8 == 2 || b8 == 4 || b8 == 8; }
bool z_b8_supported(int64_t nbw) { return nbw % 8 == 0 && nbw >= 8 && nbw <= 128; }

bool z_shape_compiled(int b8, int D, int CW, int NZ) {
    if (z_full_menu(b8)) {
        for (const ZShape &s : kZShapes)
            if (s.D == D && s.CW == CW && s.NZ == NZ) return true;
        return false;
    }
    for (const ZShape &s : kZSmallShapes)
        if (s.D == D && s.CW == CW && s.NZ == NZ) return true;
    return false;
}

struct ZPlan {
    int kernel = ELPA_B200_KERNEL_REFERENCE;
    int b8 = 0, D = 1, CW = 1, NZ = 1, K = 1;
    int grid_req = 0;
    int64_t items = 0, grid = 1;
    int threads = 128;
    size_t smem = 0;
    int64_t ws_bytes = 0;
};

size_t z_smem(int b8, int D, int CW, int NZ) {
    const size_t blob = size_t(blob_doubles(b8 + 1, 2)) * 8;
    const int stages = (D * blob * 3 <= 100 * 1024) ? 3 : 2;
    return size_t(stages) * D * blob + size_t(2) * D * CW * (2 * NZ) * 64 * 8 + size_t(2) * CW * (2 * NZ) * 64 * 8 + 64;
}

int z_make_plan(int64_t n, int64_t nbw, int64_t nev, const elpa_b200_opts *o, ZPlan &p) {
    int kernel = o ? o->kernel : ELPA_B200_KERNEL_AUTO;
    if (o && o->fused_k) return ELPA_B200_ERR_ARG;          // a DFMA-kernel knob
    if (kernel != ELPA_B200_KERNEL_AUTO && kernel != ELPA_B200_KERNEL_REFERENCE && kernel != ELPA_B200_KERNEL_DMMA)
        return ELPA_B200_ERR_ARG;
    if (kernel == ELPA_B200_KERNEL_AUTO)
        kernel = z_b8_supported(nbw) ? ELPA_B200_KERNEL_DMMA : ELPA_B200_KERNEL_REFERENCE;
    if (kernel == ELPA_B200_KERNEL_DMMA && !z_b8_supported(nbw)) return ELPA_B200_ERR_ARG;
    p.kernel = kernel;
    if (kernel == ELPA_B200_KERNEL_REFERENCE) {
        p.threads = 128;
        p.grid = (nev + 127) / 128;
        return ELPA_B200_OK;
    }
    p.b8 = int(nbw / 8);
    int D = o ? o->depth_warps : 0, CW = o ? o->col_warps : 0, NZ = o ? o->tiles_per_warp : 0;
    int K = (o && o->groups_per_step) ? o->groups_per_step : 0;
    const int64_t ntile_z = (nev + 7) / 8;
    if (D == 0 && CW == 0 && NZ == 0 && K == 0 && (p.b8 == 8 || p.b8 == 4) && ntile_z < 1000) {
        // thin complex stripes run the two-group register window (kernel_dmma_kwin.cuh):
        // 2000 columns 29.2 TF/s against 28.3, 5000 30.0 against 29.8; at 20000 the K = 1 kernel
        // stays ahead, 30.7 against 30.3 (profiles/r02/c64_kwin_r02.jsonl); nbw = 32: C2 25.9
        // against 24.6, 20000 x 2000 26.2 against 24.9 (c64_kwin_nbw32_r02.log)
        D = 1; CW = 4; NZ = 1; K = 2;
    }
    if (K == 0) K = 1;
    if (D == 0 && CW == 0 && NZ == 0) {
        // (1,4,1) everywhere on the full menu: MEDIUM autotuning with the ring-mode kernel
        // (profiles/autotune_medium_r01_final.jsonl) picks it at C4 (28.2 TF/s; (2,2,2) measured
        // 22.1) and keeps the automatic choice at C2; C3 (1,4,1) 30.7
        if (z_full_menu(p.b8)) { D = 1; CW = 4; NZ = 1; }
        else { D = 2; CW = 2; NZ = 1; }
    }
    const bool kwin = K >= 2;
    if (kwin ? !zk_compiled(p.b8, D, CW, NZ, K) : !z_shape_compiled(p.b8, D, CW, NZ)) return ELPA_B200_ERR_ARG;
    p.D = D; p.CW = CW; p.NZ = NZ; p.K = K;
    p.grid_req = o ? o->grid_ctas : 0;
    if (p.grid_req < 0) return ELPA_B200_ERR_ARG;
    const int64_t M = num_depths(n, nbw);
    const int64_t ntile = (nev + 7) / 8;
    const int64_t nx = (ntile + CW * NZ - 1) / (CW * NZ);
    p.items = nx * ((M + D - 1) / D);
    p.grid = p.items;
    p.threads = 32 * D * CW;
    p.smem = kwin ? kwin_smem(p.b8, CW, 2 * NZ, K, kwin_stages(p.b8, CW, 2 * NZ, K, KIND_ZMMA), KIND_ZMMA)
                  : z_smem(p.b8, D, CW, NZ);
    if (p.smem > size_t(smem_optin())) return ELPA_B200_ERR_ARG;
    p.ws_bytes = (M > 0) ? total_groups(n, p.b8, M) * blob_doubles(p.b8 + 1, 2) * 8 : 0;
    return ELPA_B200_OK;
}

int z_validate(int64_t n, int64_t nbw, int64_t nev, const void *hh_v, const void *hh_tau, const void *Q, int64_t ldq) {
    if (n < 0 || nbw < 1 || nev < 0 || nev > n || ldq < (n > 1 ? n : 1) || n > kMaxN) return ELPA_B200_ERR_ARG;
    const int64_t R = hh_total(n, nbw);
    if (R > 0 && nev > 0 && (!hh_v || !hh_tau || !Q)) return ELPA_B200_ERR_NULL;
    if (R > 0 && nev > 0 && (reinterpret_cast<uintptr_t>(Q) & 15)) return ELPA_B200_ERR_ALIGN;
    return ELPA_B200_OK;
}

template <int B8, int D, int CW, int NZ>
int z_launch_shape(const ZPlan &p, int64_t n, int64_t nev, const double *ws, double *Q, int64_t ldq, cudaStream_t s) {
    using Cfg = DmmaCfg<KIND_ZMMA, B8, D, CW, 2 * NZ, 1>;
    auto kern = apply_dmma_kernel<KIND_ZMMA, B8, D, CW, 2 * NZ, 1>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM)) != cudaSuccess)
        return fail_cuda();
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::THREADS, Cfg::SMEM) != cudaSuccess ||
        per_sm < 1)
        return fail_cuda();
    int64_t grid = int64_t(per_sm) * sm_count();
    if (p.grid_req > 0 && p.grid_req < grid) grid = p.grid_req;
    if (grid > p.items) grid = p.items;
    uint64_t *prog = nullptr;
    const size_t pbytes = size_t(p.items + 1) * 8;
    if (lib_malloc_async(reinterpret_cast<void **>(&prog), pbytes, s) != cudaSuccess) return fail_cuda();
    int rc = ELPA_B200_OK;
    if (cudaMemsetAsync(prog, 0, pbytes, s) != cudaSuccess) rc = ELPA_B200_ERR_CUDA;
    if (rc == ELPA_B200_OK) {
        kern<<<unsigned(grid), Cfg::THREADS, Cfg::SMEM, s>>>(n, nev, ws, Q, ldq, prog, pub_period());
        if (cudaGetLastError() != cudaSuccess) rc = ELPA_B200_ERR_CUDA;
    }
    if (cudaFreeAsync(prog, s) != cudaSuccess && rc == ELPA_B200_OK) rc = ELPA_B200_ERR_CUDA;
    return rc;
}

template <int B8, int CW, int NZ, int K>
int zk_launch_shape(const ZPlan &p, int64_t n, int64_t nev, const double *ws, double *Q, int64_t ldq, cudaStream_t s) {
    using Cfg = KwinCfg<B8, CW, 2 * NZ, K, KIND_ZMMA>;
    auto kern = apply_dmma_kwin_kernel<B8, CW, 2 * NZ, K, KIND_ZMMA>;
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
int z_run_b8(const ZPlan &p, int64_t n, int64_t nev, const double *hh_v, const double *hh_tau, double *ws, double *Q,
             int64_t ldq, cudaStream_t s) {
    const int64_t M = num_depths(n, 8 * B8);
    const int64_t G0 = groups_at_depth(n, B8, 0);
    prep_zmma_kernel<B8><<<dim3(unsigned((G0 + 1) / 2), unsigned(M)), 64, 0, s>>>(n, hh_v, hh_tau, ws);
    if (cudaGetLastError() != cudaSuccess) return ELPA_B200_ERR_CUDA;
    if constexpr (B8 == 4 || B8 == 8) {
#define ELPA_ZK_CASE(CW_, NZ_, K_) \
        if (p.K == K_ && p.CW == CW_ && p.NZ == NZ_) return zk_launch_shape<B8, CW_, NZ_, K_>(p, n, nev, ws, Q, ldq, s);
        ELPA_ZK_SHAPES(ELPA_ZK_CASE)
#undef ELPA_ZK_CASE
    }
    if (p.K != 1) return ELPA_B200_ERR_ARG;
#define ELPA_Z_CASE(D_, CW_, NZ_) \
    if (p.D == D_ && p.CW == CW_ && p.NZ == NZ_) return z_launch_shape<B8, D_, CW_, NZ_>(p, n, nev, ws, Q, ldq, s);
    if constexpr (B8 == 1 || B8 == 2 || B8 == 4 || B8 == 8) {
        ELPA_Z_SHAPES(ELPA_Z_CASE)
    } else {
        ELPA_Z_SMALL_SHAPES(ELPA_Z_CASE)
    }
#undef ELPA_Z_CASE
    return ELPA_B200_ERR_ARG;
}

int z_run(const ZPlan &p, int64_t n, int64_t nbw, int64_t nev, const double *hh_v, const double *hh_tau, double *Q,
          int64_t ldq, cudaStream_t s) {
    if (p.kernel == ELPA_B200_KERNEL_REFERENCE) {
        apply_reference_c_kernel<<<unsigned(p.grid), p.threads, 0, s>>>(n, nbw, nev, hh_v, hh_tau, Q, ldq);
        return cudaGetLastError() == cudaSuccess ? ELPA_B200_OK : ELPA_B200_ERR_CUDA;
    }
    double *ws = nullptr;
    if (p.ws_bytes > 0 && lib_malloc_async(reinterpret_cast<void **>(&ws), size_t(p.ws_bytes), s) != cudaSuccess)
        return fail_cuda();
    int rc = ELPA_B200_ERR_ARG;
    switch (p.b8) {
#define ELPA_Z_B8(B8_) \
    case B8_: rc = z_run_b8<B8_>(p, n, nev, hh_v, hh_tau, ws, Q, ldq, s); break;
        ELPA_Z_B8(1) ELPA_Z_B8(2) ELPA_Z_B8(3) ELPA_Z_B8(4) ELPA_Z_B8(5) ELPA_Z_B8(6) ELPA_Z_B8(7) ELPA_Z_B8(8)
        ELPA_Z_B8(9) ELPA_Z_B8(10) ELPA_Z_B8(11) ELPA_Z_B8(12) ELPA_Z_B8(13) ELPA_Z_B8(14) ELPA_Z_B8(15)
        ELPA_Z_B8(16)
#undef ELPA_Z_B8
    }
    if (ws && cudaFreeAsync(ws, s) != cudaSuccess && rc == ELPA_B200_OK) rc = ELPA_B200_ERR_CUDA;
    return rc;
}

}  // namespace

int elpa_b200_host::c64_shape_menu(int b8, int (*out)[4], int max) {
    int k = 0;
    auto add = [&](const ZShape *sh, int cnt) {
        for (int i = 0; i < cnt && k < max; i++, k++) {
            out[k][0] = sh[i].D; out[k][1] = sh[i].CW; out[k][2] = sh[i].NZ; out[k][3] = 1;
        }
    };
    if (!z_b8_supported(8 * int64_t(b8))) return 0;
    if (z_full_menu(b8)) add(kZShapes, int(sizeof(kZShapes) / sizeof(kZShapes[0])));
    else add(kZSmallShapes, int(sizeof(kZSmallShapes) / sizeof(kZSmallShapes[0])));
    if (b8 == 4 || b8 == 8)                              // the register-window shapes (K = 2)
        for (const ZkShape &z : kZkShapes)
            if (k < max) {
                out[k][0] = 1; out[k][1] = z.CW; out[k][2] = z.NZ; out[k][3] = z.K;
                k++;
            }
    return k;
}

extern "C" {

int elpa_trans_ev_tridi_to_band_c64(int64_t n, int64_t nbw, int64_t nev, const double *hh_v, const double *hh_tau,
                                    double *Q, int64_t ldq, elpa_b200_stream_t stream, const elpa_b200_opts *opts) {
    int rc = z_validate(n, nbw, nev, hh_v, hh_tau, Q, ldq);
    if (rc != ELPA_B200_OK) return rc;
    ZPlan p;
    if ((rc = z_make_plan(n, nbw, nev, opts, p)) != ELPA_B200_OK) return rc;
    if (hh_total(n, nbw) == 0 || nev == 0) return ELPA_B200_OK;
    if ((rc = check_device()) != ELPA_B200_OK) return rc;
    return z_run(p, n, nbw, nev, hh_v, hh_tau, Q, ldq, reinterpret_cast<cudaStream_t>(stream));
}

int elpa_b200_describe_c64(int64_t n, int64_t nbw, int64_t nev, const elpa_b200_opts *opts, char *buf,
                           size_t buflen) {
    if (n < 0 || nbw < 1 || nev < 0 || nev > n) return ELPA_B200_ERR_ARG;
    ZPlan p;
    int rc = z_make_plan(n, nbw, nev, opts, p);
    if (rc != ELPA_B200_OK) return rc;
    if (buf && buflen)
        snprintf(buf, buflen, "kernel=%s b8=%d D=%d CW=%d NZ=%d K=%d items=%lld grid_req=%d block=%d smem=%zu ws=%lld",
                 p.kernel == ELPA_B200_KERNEL_DMMA ? "zmma" : "reference_c64", p.b8, p.D, p.CW, p.NZ, p.K,
                 (long long)p.items, p.grid_req, p.threads, p.smem, (long long)p.ws_bytes);
    if (hh_total(n, nbw) == 0 || nev == 0) return 0;
    return p.kernel == ELPA_B200_KERNEL_REFERENCE ? 1 : 2;
}

}  // extern "C"
