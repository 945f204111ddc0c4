// elpa_b200_f32.cu — C-ABI entry points of the FP32 variant of the hot path (SURVEY §8f NEXT-3,
// include/elpa_b200.h "FP32 variant"): validation, plan, reflector preparation and launch of
// apply_f32_kernel (kernel_f32.cuh).  Same operation and conventions as the FP64 path.
#include <cuda_runtime.h>

#include <cstdio>

#include "../../include/elpa_b200.h"
#include "geometry.cuh"
#include "host_common.h"
#include "kernel_f32.cuh"

using namespace elpa_b200;
using namespace elpa_b200_host;

namespace {

// (D depth warps, CW column warps, NC 32-column blocks per warp, K groups per step) menus.
// Full menu for nbw = 8/16/32/64, a small one for the other multiples of 8 up to 128
// (compile-time budget).
#define ELPA_F32_SHAPES(X) X(1, 2, 1, 1) X(2, 2, 1, 1) X(1, 4, 1, 1) X(2, 1, 1, 1) X(4, 2, 1, 1) X(1, 1, 2, 1) \
    X(1, 2, 2, 1) X(2, 1, 2, 1) X(1, 1, 1, 1) X(1, 2, 1, 2) X(2, 2, 1, 2) X(2, 1, 1, 2)
#define ELPA_F32_SMALL_SHAPES(X) X(1, 2, 1, 1) X(2, 2, 1, 1)
struct F32Shape { int D, CW, NC, K; };
#define ELPA_F32_ENTRY(D_, CW_, NC_, K_) {D_, CW_, NC_, K_},
constexpr F32Shape kF32Shapes[] = {ELPA_F32_SHAPES(ELPA_F32_ENTRY)};
constexpr F32Shape kF32SmallShapes[] = {ELPA_F32_SMALL_SHAPES(ELPA_F32_ENTRY)};

bool f32_full_menu(int b8) { return b8 == 1 || b8 == 2 || b8 == 4 || b8 == 8; }
bool f32_b8_supported(int64_t nbw) { return nbw % 8 == 0 && nbw >= 8 && nbw <= 128; }

bool f32_shape_compiled(int b8, int D, int CW, int NC, int K) {
    if (f32_full_menu(b8)) {
        for (const F32Shape &s : kF32Shapes)
            if (s.D == D && s.CW == CW && s.NC == NC && s.K == K) return true;
        return false;
    }
    for (const F32Shape &s : kF32SmallShapes)
        if (s.D == D && s.CW == CW && s.NC == NC && s.K == K) return true;
    return false;
}

size_t f32_smem(int b8, int D, int CW, int NC, int K) {
    const size_t blob = size_t(f32_blob_floats(b8)) * 4;
    const int stages = (K * D * blob * 3 <= 100 * 1024) ? 3 : 2;
    return size_t(stages) * K * D * blob + size_t(2) * D * K * CW * NC * 2 * 32 * 16 +
           size_t(2) * K * CW * NC * 2 * 32 * 16 + 64;
}

struct F32Plan {
    int kernel = ELPA_B200_KERNEL_REFERENCE;
    int b8 = 0, D = 1, CW = 1, NC = 1, K = 1;
    int grid_req = 0;
    int64_t items = 0, nx = 0, grid = 1;
    int threads = 128;
    size_t smem = 0;
    int64_t ws_bytes = 0;
};

int f32_make_plan(int64_t n, int64_t nbw, int64_t nev, const elpa_b200_opts *o, F32Plan &p) {
    int kernel = o ? o->kernel : ELPA_B200_KERNEL_AUTO;
    if (o && o->fused_k) return ELPA_B200_ERR_ARG;          // a DFMA-kernel knob
    if (kernel != ELPA_B200_KERNEL_AUTO && kernel != ELPA_B200_KERNEL_REFERENCE && kernel != ELPA_B200_KERNEL_FFMA2)
        return ELPA_B200_ERR_ARG;
    if (kernel == ELPA_B200_KERNEL_AUTO)
        kernel = f32_b8_supported(nbw) ? ELPA_B200_KERNEL_FFMA2 : ELPA_B200_KERNEL_REFERENCE;
    if (kernel == ELPA_B200_KERNEL_FFMA2 && !f32_b8_supported(nbw)) return ELPA_B200_ERR_ARG;
    p.kernel = kernel;
    if (kernel == ELPA_B200_KERNEL_REFERENCE) {
        p.threads = 128;
        p.grid = (nev + 127) / 128;
        return ELPA_B200_OK;
    }
    p.b8 = int(nbw / 8);
    int D = o ? o->depth_warps : 0, CW = o ? o->col_warps : 0, NC = o ? o->tiles_per_warp : 0;
    int K = o ? o->groups_per_step : 0;
    if (D == 0 && CW == 0 && NC == 0) { D = 2; CW = 2; NC = 1; }
    if (K == 0) K = 1;
    if (!f32_shape_compiled(p.b8, D, CW, NC, K)) return ELPA_B200_ERR_ARG;
    p.D = D; p.CW = CW; p.NC = NC; p.K = K;
    p.grid_req = o ? o->grid_ctas : 0;
    if (p.grid_req < 0) return ELPA_B200_ERR_ARG;
    const int64_t M = num_depths(n, nbw);
    const int64_t cols = int64_t(CW) * NC * 32;
    p.nx = (nev + cols - 1) / cols;
    p.items = p.nx * ((M + D - 1) / D);
    p.grid = p.items;
    p.threads = 32 * D * CW;
    p.smem = f32_smem(p.b8, D, CW, NC, K);
    if (p.smem > size_t(smem_optin())) return ELPA_B200_ERR_ARG;
    p.ws_bytes = (M > 0) ? total_groups(n, p.b8, M) * f32_blob_floats(p.b8) * 4 : 0;
    return ELPA_B200_OK;
}

int f32_validate(int64_t n, int64_t nbw, int64_t nev, const void *hh_v, const void *hh_tau, const void *Q,
                 int64_t ldq) {
    if (n < 0 || nbw < 1 || nev < 0 || nev > n || ldq < (n > 1 ? n : 1) || n > kMaxN) return ELPA_B200_ERR_ARG;
    const int64_t R = hh_total(n, nbw);
    if (R > 0 && nev > 0 && (!hh_v || !hh_tau || !Q)) return ELPA_B200_ERR_NULL;
    if (R > 0 && nev > 0 && ((ldq & 3) || (reinterpret_cast<uintptr_t>(Q) & 15))) return ELPA_B200_ERR_ALIGN;
    return ELPA_B200_OK;
}

template <int B8>
int f32_launch_prep(int64_t n, const float *hh_v, const float *hh_tau, float *ws, cudaStream_t s) {
    const int64_t M = num_depths(n, 8 * B8);
    const int64_t G0 = groups_at_depth(n, B8, 0);
    dim3 grid(unsigned((G0 + 7) / 8), unsigned(M));
    prep_f32_kernel<B8><<<grid, 256, 0, s>>>(n, hh_v, hh_tau, ws);
    return cudaGetLastError() == cudaSuccess ? ELPA_B200_OK : ELPA_B200_ERR_CUDA;
}

template <int B8, int D, int CW, int NC, int K>
int f32_launch_shape(const F32Plan &p, int64_t n, int64_t nev, const float *ws, float *Q, int64_t ldq,
                     cudaStream_t s) {
    using Cfg = F32Cfg<B8, D, CW, NC, K>;
    auto kern = apply_f32_kernel<B8, D, CW, NC, K>;
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

template <int B8>
int f32_launch_b8(const F32Plan &p, int64_t n, int64_t nev, const float *ws, float *Q, int64_t ldq, cudaStream_t s) {
#define ELPA_F32_CASE(D_, CW_, NC_, K_)                               \
    if (p.D == D_ && p.CW == CW_ && p.NC == NC_ && p.K == K_) \
        return f32_launch_shape<B8, D_, CW_, NC_, K_>(p, n, nev, ws, Q, ldq, s);
    if constexpr (B8 == 1 || B8 == 2 || B8 == 4 || B8 == 8) {
        ELPA_F32_SHAPES(ELPA_F32_CASE)
    } else {
        ELPA_F32_SMALL_SHAPES(ELPA_F32_CASE)
    }
#undef ELPA_F32_CASE
    return ELPA_B200_ERR_ARG;
}

int f32_run(const F32Plan &p, int64_t n, int64_t nbw, int64_t nev, const float *hh_v, const float *hh_tau, float *Q,
            int64_t ldq, cudaStream_t s) {
    if (p.kernel == ELPA_B200_KERNEL_REFERENCE) {
        apply_reference_f32_kernel<<<unsigned(p.grid), p.threads, 0, s>>>(n, nbw, nev, hh_v, hh_tau, Q, ldq);
        return cudaGetLastError() == cudaSuccess ? ELPA_B200_OK : ELPA_B200_ERR_CUDA;
    }
    float *ws = nullptr;
    if (p.ws_bytes > 0 && lib_malloc_async(reinterpret_cast<void **>(&ws), size_t(p.ws_bytes), s) != cudaSuccess)
        return fail_cuda();
    int rc = ELPA_B200_ERR_ARG;
    switch (p.b8) {
#define ELPA_F32_B8(B8_)                                                 \
    case B8_:                                                            \
        rc = f32_launch_prep<B8_>(n, hh_v, hh_tau, ws, s);               \
        if (rc == ELPA_B200_OK) rc = f32_launch_b8<B8_>(p, n, nev, ws, Q, ldq, s); \
        break;
        ELPA_F32_B8(1) ELPA_F32_B8(2) ELPA_F32_B8(3) ELPA_F32_B8(4) ELPA_F32_B8(5) ELPA_F32_B8(6) ELPA_F32_B8(7)
        ELPA_F32_B8(8) ELPA_F32_B8(9) ELPA_F32_B8(10) ELPA_F32_B8(11) ELPA_F32_B8(12) ELPA_F32_B8(13)
        ELPA_F32_B8(14) ELPA_F32_B8(15) ELPA_F32_B8(16)
#undef ELPA_F32_B8
    }
    if (ws && cudaFreeAsync(ws, s) != cudaSuccess && rc == ELPA_B200_OK) rc = ELPA_B200_ERR_CUDA;
    return rc;
}

}  // namespace

int elpa_b200_host::f32_shape_menu(int b8, int (*out)[4], int max) {
    int k = 0;
    auto add = [&](const F32Shape *sh, int cnt) {
        for (int i = 0; i < cnt && k < max; i++, k++) {
            out[k][0] = sh[i].D; out[k][1] = sh[i].CW; out[k][2] = sh[i].NC; out[k][3] = sh[i].K;
        }
    };
    if (!f32_b8_supported(8 * int64_t(b8))) return 0;
    if (f32_full_menu(b8)) add(kF32Shapes, int(sizeof(kF32Shapes) / sizeof(kF32Shapes[0])));
    else add(kF32SmallShapes, int(sizeof(kF32SmallShapes) / sizeof(kF32SmallShapes[0])));
    return k;
}

extern "C" {

int elpa_trans_ev_tridi_to_band_f32(int64_t n, int64_t nbw, int64_t nev, const float *hh_v, const float *hh_tau,
                                    float *Q, int64_t ldq, elpa_b200_stream_t stream, const elpa_b200_opts *opts) {
    int rc = f32_validate(n, nbw, nev, hh_v, hh_tau, Q, ldq);
    if (rc != ELPA_B200_OK) return rc;
    F32Plan p;
    if ((rc = f32_make_plan(n, nbw, nev, opts, p)) != ELPA_B200_OK) return rc;
    if (hh_total(n, nbw) == 0 || nev == 0) return ELPA_B200_OK;
    if ((rc = check_device()) != ELPA_B200_OK) return rc;
    return f32_run(p, n, nbw, nev, hh_v, hh_tau, Q, ldq, reinterpret_cast<cudaStream_t>(stream));
}

int elpa_b200_describe_f32(int64_t n, int64_t nbw, int64_t nev, const elpa_b200_opts *opts, char *buf,
                           size_t buflen) {
    if (n < 0 || nbw < 1 || nev < 0 || nev > n) return ELPA_B200_ERR_ARG;
    F32Plan p;
    int rc = f32_make_plan(n, nbw, nev, opts, p);
    if (rc != ELPA_B200_OK) return rc;
    if (buf && buflen)
        snprintf(buf, buflen, "kernel=%s b8=%d D=%d CW=%d NC=%d K=%d items=%lld grid_req=%d block=%d smem=%zu ws=%lld",
                 p.kernel == ELPA_B200_KERNEL_FFMA2 ? "ffma2" : "reference_f32", p.b8, p.D, p.CW, p.NC, p.K,
                 (long long)p.items, p.grid_req, p.threads, p.smem, (long long)p.ws_bytes);
    if (hh_total(n, nbw) == 0 || nev == 0) return 0;
    return p.kernel == ELPA_B200_KERNEL_REFERENCE ? 1 : 2;
}

}  // extern "C"
