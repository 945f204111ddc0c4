// elpa_b200_dense.cu — C-ABI entry points of the dense steps next to the hot path:
// NEXT-1 elpa_trans_ev_band_to_full and NEXT-4 elpa_generalized_back_transform
// (Eq. 7).  Every product runs in the library's own FP64 tensor-core contraction
// (dgemm_dmma.cuh); the preparation kernels are band_to_full.cuh / gen_back.cuh.  No BLAS.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/elpa_b200.h"
#include "host_common.h"
#include "dgemm_host.h"
#include "band_to_full.cuh"
#include "gen_back.cuh"

using namespace elpa_b200;
using namespace elpa_b200_host;

namespace {

// Panel width: the Q update's reduction length.  512 measured 0.88 of the DMMA peak for the update
// and 0.91 for V^T Q against 0.84 / 0.89 at 256 (tools/gemm_bench.cu); the G and U products it adds
// cost 2.6% of the flops.
constexpr int64_t kB2FPanel = 512;

size_t up256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

extern "C" {

int64_t elpa_b2f_count(int64_t n, int64_t nbw) {
    if (n < 0 || nbw < 1) return -1;
    return n >= nbw + 2 ? n - nbw - 1 : 0;
}

int elpa_trans_ev_band_to_full(int64_t n, int64_t nbw, int64_t nev, const double *hh1_v, int64_t ldv,
                               const double *hh1_tau, double *Q, int64_t ldq, elpa_b200_stream_t stream) {
    if (n < 0 || nbw < 1 || nev < 0 || nev > n || ldq < (n > 1 ? n : 1) || ldv < (n > 1 ? n : 1) || n > kMaxN)
        return ELPA_B200_ERR_ARG;
    const int64_t K = elpa_b2f_count(n, nbw);
    if (K == 0 || nev == 0) return ELPA_B200_OK;
    if (!hh1_v || !hh1_tau || !Q) return ELPA_B200_ERR_NULL;
    int rc = check_device();
    if (rc != ELPA_B200_OK) return rc;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t P = kB2FPanel, np = (K + P - 1) / P;
    const int64_t m0 = b2f_rows(n, nbw, P, 0), ld0 = b2f_ld(n, nbw, P, 0);
    // workspace: V panels and U^T panels (same size), G and T per panel, one panel's V^T, W^T,
    // and the split-K partials of the largest product of each kind
    const size_t nV = size_t(b2f_panel_offset(n, nbw, P, np));
    size_t nScr = 0, nCnt = 0;
    for (int64_t p = 0; p < np; p++) {
        const int64_t m = b2f_rows(n, nbw, P, p);
        nCnt = std::max<size_t>({nCnt, size_t(gemm_tiles(m, P)), size_t(gemm_tiles(nev, P)), size_t(gemm_tiles(nev, m))});
        nScr = std::max<size_t>(nScr, size_t(gemm_scratch_doubles(P, P, m)));        // G
        nScr = std::max<size_t>(nScr, size_t(gemm_scratch_doubles(m, P, P)));        // U^T
        nScr = std::max<size_t>(nScr, size_t(gemm_scratch_doubles(nev, P, m)));      // W^T
        nScr = std::max<size_t>(nScr, size_t(gemm_scratch_doubles(nev, m, P)));      // Q update
    }
    const size_t bV = up256(nV * 8), bG = up256(size_t(np) * P * P * 8), bVT = up256(size_t(ld0) * P * 8);
    const size_t bW = up256(size_t(nev) * P * 8), bS = up256(nScr * 8), bC = up256(nCnt * 4);
    char *buf = nullptr;
    if (lib_malloc_async(reinterpret_cast<void **>(&buf), 2 * bV + 2 * bG + bVT + bW + bS + bC, s) != cudaSuccess)
        return fail_cuda();
    unsigned *cnt = reinterpret_cast<unsigned *>(buf + 2 * bV + 2 * bG + bVT + bW + bS);
    if (cudaMemsetAsync(cnt, 0, nCnt * 4, s) != cudaSuccess) rc = ELPA_B200_ERR_CUDA;
    double *Vp = reinterpret_cast<double *>(buf), *UT = reinterpret_cast<double *>(buf + bV);
    double *G = reinterpret_cast<double *>(buf + 2 * bV), *T = reinterpret_cast<double *>(buf + 2 * bV + bG);
    double *VT = reinterpret_cast<double *>(buf + 2 * bV + 2 * bG);
    double *Wt = reinterpret_cast<double *>(buf + 2 * bV + 2 * bG + bVT);
    double *scr = reinterpret_cast<double *>(buf + 2 * bV + 2 * bG + bVT + bW);
    (void)m0;
    if (rc == ELPA_B200_OK) {
        dim3 g(unsigned(std::min<int64_t>(1024, (ld0 * P + 255) / 256)), unsigned(np));
        b2f_build_panels<<<g, 256, 0, s>>>(n, nbw, K, P, hh1_v, ldv, Vp);
        if (cudaGetLastError() != cudaSuccess) rc = ELPA_B200_ERR_CUDA;
    }
    // G_p = V_p^T V_p, then T_p (dlarft), then U_p^T = -(V_p T_p)^T stored row-major per row
    for (int64_t p = 0; rc == ELPA_B200_OK && p < np; p++) {
        const int64_t ld = b2f_ld(n, nbw, P, p);
        const double *vp = Vp + b2f_panel_offset(n, nbw, P, p);
        // G_p = V_p^T V_p: column a of V_p is zero above relative row a (the staircase)
        rc = gemm_tn(P, P, ld, 1.0, vp, ld, vp, ld, 0.0, G + p * P * P, P, scr, cnt, s, GEMM_A_STAIR | GEMM_B_STAIR);
    }
    if (rc == ELPA_B200_OK) {
        static bool attr = cudaFuncSetAttribute(b2f_tfactor, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                int(kTfactorSmem)) == cudaSuccess;
        if (!attr) rc = ELPA_B200_ERR_CUDA;
        else b2f_tfactor<<<unsigned(np), 512, kTfactorSmem, s>>>(K, P, hh1_tau, G, T);
        if (cudaGetLastError() != cudaSuccess) rc = ELPA_B200_ERR_CUDA;
    }
    for (int64_t p = 0; rc == ELPA_B200_OK && p < np; p++) {
        const int64_t ld = b2f_ld(n, nbw, P, p), off = b2f_panel_offset(n, nbw, P, p);
        dim3 g(unsigned((ld + 31) / 32), unsigned((P + 31) / 32));
        b2f_transpose_panel<<<g, 256, 0, s>>>(ld, ld, P, Vp + off, VT);
        if (cudaGetLastError() != cudaSuccess) { rc = ELPA_B200_ERR_CUDA; break; }
        // UT[i*P + c] = -sum_a V[i][a] T[a][c]:  A = V^T (K = a, M = i), B = T (K = a, N = c)
        rc = gemm_tn(ld, P, P, -1.0, VT, P, T + p * P * P, P, 0.0, UT + off, P, scr, cnt, s, GEMM_B_UPPER);
    }
    // apply, last panel first:  W^T = Q^T V_p,  Q^T += W^T U_p^T  (rows r0' .. n of Q)
    for (int64_t p = np - 1; rc == ELPA_B200_OK && p >= 0; p--) {
        const int64_t r0 = b2f_origin(nbw, P, p), m = n - r0, ld = b2f_ld(n, nbw, P, p);
        const int64_t off = b2f_panel_offset(n, nbw, P, p);
        rc = gemm_tn(nev, P, m, 1.0, Q + r0, ldq, Vp + off, ld, 0.0, Wt, P, scr, cnt, s, GEMM_B_STAIR);
        if (rc == ELPA_B200_OK) rc = gemm_tn(nev, m, P, 1.0, Wt, P, UT + off, P, 1.0, Q + r0, ldq, scr, cnt, s);
    }
    if (cudaFreeAsync(buf, s) != cudaSuccess && rc == ELPA_B200_OK) rc = ELPA_B200_ERR_CUDA;
    if (rc != ELPA_B200_OK) cudaGetLastError();
    return rc;
}

int elpa_generalized_back_transform(int64_t n, int64_t nev, const double *L, int64_t ldl, double *Q, int64_t ldq,
                                    elpa_b200_stream_t stream) {
    if (n < 0 || nev < 0 || nev > n || ldl < (n > 1 ? n : 1) || ldq < (n > 1 ? n : 1) || n > kMaxN)
        return ELPA_B200_ERR_ARG;
    if (n == 0 || nev == 0) return ELPA_B200_OK;
    if (!L || !Q) return ELPA_B200_ERR_NULL;
    int rc = check_device();
    if (rc != ELPA_B200_OK) return rc;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    constexpr int NB = kGbBlock;
    const int64_t nb = (n + NB - 1) / NB;
    size_t nScr = 0;
    const size_t nCnt = size_t(gemm_tiles(nev, NB));
    for (int64_t b = 0; b < nb; b++) {
        const int64_t r1 = std::min<int64_t>(n, (b + 1) * NB);
        nScr = std::max<size_t>(nScr, size_t(gemm_scratch_doubles(nev, NB, n - r1)));
        nScr = std::max<size_t>(nScr, size_t(gemm_scratch_doubles(nev, NB, NB)));
    }
    const size_t bInv = up256(size_t(nb) * NB * NB * 8), bT = up256(size_t(NB) * nev * 8), bS = up256(nScr * 8);
    char *buf = nullptr;
    if (lib_malloc_async(reinterpret_cast<void **>(&buf), bInv + bT + bS + up256(nCnt * 4), s) != cudaSuccess)
        return fail_cuda();
    unsigned *cnt = reinterpret_cast<unsigned *>(buf + bInv + bT + bS);
    if (cudaMemsetAsync(cnt, 0, nCnt * 4, s) != cudaSuccess) rc = ELPA_B200_ERR_CUDA;
    double *Linv = reinterpret_cast<double *>(buf), *T = reinterpret_cast<double *>(buf + bInv);
    double *scr = reinterpret_cast<double *>(buf + bInv + bT);
    const size_t smem = size_t(NB) * NB * 8;
    if (rc == ELPA_B200_OK &&
        cudaFuncSetAttribute(gb_trinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
        rc = ELPA_B200_ERR_CUDA;
    if (rc == ELPA_B200_OK) {
        gb_trinv_kernel<<<unsigned(nb), NB, smem, s>>>(n, L, ldl, Linv);
        if (cudaGetLastError() != cudaSuccess) rc = ELPA_B200_ERR_CUDA;
    }
    // left-looking from the bottom: Q_b -= L[r1:n, r0:r1]^T Q[r1:n];  Q_b = L_bb^{-T} Q_b
    for (int64_t b = nb - 1; rc == ELPA_B200_OK && b >= 0; b--) {
        const int64_t r0 = b * NB, m = std::min<int64_t>(NB, n - r0), r1 = r0 + m;
        if (r1 < n) rc = gemm_tn(nev, m, n - r1, -1.0, Q + r1, ldq, L + r0 * ldl + r1, ldl, 1.0, Q + r0, ldq, scr, cnt, s);
        // T[c*NB + i] = sum_k Q_b[k][c] Linv[k][i]  (Linv column-major, ld NB)
        // (L_bb^{-1} is lower triangular: column i of B is zero above row i)
        if (rc == ELPA_B200_OK)
            rc = gemm_tn(nev, m, m, 1.0, Q + r0, ldq, Linv + b * NB * NB, NB, 0.0, T, NB, scr, cnt, s, GEMM_B_STAIR);
        if (rc == ELPA_B200_OK &&
            cudaMemcpy2DAsync(Q + r0, size_t(ldq) * 8, T, size_t(NB) * 8, size_t(m) * 8, size_t(nev),
                              cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            rc = ELPA_B200_ERR_CUDA;
    }
    if (cudaFreeAsync(buf, s) != cudaSuccess && rc == ELPA_B200_OK) rc = ELPA_B200_ERR_CUDA;
    if (rc != ELPA_B200_OK) cudaGetLastError();
    return rc;
}

}  // extern "C"
