// host_common.h — host-side helpers shared by the library's translation units
// (elpa_b200.cu: FP64 path, elpa_b200_f32.cu: FP32 path).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "../../include/elpa_b200.h"

namespace elpa_b200_host {

constexpr int kMaxSms = 148;
// The kernels index rows and chunks with 32-bit integers (row 8c + 7 < 2^31).
constexpr int64_t kMaxN = (int64_t(1) << 31) - 64;

inline int sm_count() {
    int dev = 0, n = kMaxSms;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cudaGetLastError();
    return n > 0 ? n : kMaxSms;
}

// A failed runtime call leaves a "last error" that a later cudaGetLastError() after a
// successful launch would report; clear it so every call reports only its own failures.
inline int fail_cuda() {
    cudaGetLastError();
    return ELPA_B200_ERR_CUDA;
}

// Progress-publish period in steps: each publish is a release fence on the
// CTA's critical path, but a next pass chained right behind waits for it.  Thin column stripes
// (fewer than 2000 8-column tiles) are bound by the chain of depth passes, so they publish every
// 16 steps (measured +0.5-1% at 2000-5000 columns), wide ones every 32.  Development override:
// ELPA_B200_PUB.
inline int pub_period(int64_t ntile = 1 << 30) {
    static int v = [] {
        const char *e = getenv("ELPA_B200_PUB");
        int x = e ? atoi(e) : 0;
        return x >= 1 ? x : 0;
    }();
    if (v) return v;
    return ntile < 2000 ? 16 : 32;
}

// The register-window kernel (K groups per step) measured its own optimum
// (profiles/r02/kwin_pub_period_r02.jsonl, profiles/r02/kwin_thin_pub_r02.jsonl): 32 steps for wide
// stripes, 16 from 400 tiles, 8 below (2500 columns: 27.43 TF/s at 8 against 27.18 at 16).
inline int kwin_pub_period(int64_t ntile) {
    const int v = pub_period();
    if (v != 32) return v;                      // ELPA_B200_PUB override
    return ntile < 400 ? 8 : (ntile < 2000 ? 16 : 32);
}

inline int smem_optin() {
    int dev = 0, v = 232448;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaGetLastError();   // no device (CPU host): keep the B200 value, clear the error
    return v > 0 ? v : 232448;
}

inline int check_device() {
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return ELPA_B200_ERR_DEVICE;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
        return ELPA_B200_ERR_DEVICE;
    return (major == 10 && minor == 0) ? ELPA_B200_OK : ELPA_B200_ERR_DEVICE;
}

// The library's own stream-ordered memory pool, one per device, that keeps freed memory cached
// (release threshold = max): workspaces of several GB are then re-used across calls instead of
// being unmapped at every synchronisation and re-mapped by the next call (measured: up to
// ~190 ms per C3 call through the default pool).  elpa_b200_release_cache() trims it.
// This caching is a documented deviation from SURVEY §8(b)'s "no persistent allocation"
// (DESIGN.md §4): elpa_b200_set_workspace_cache(0) makes the pool return freed memory at every
// synchronisation (release threshold 0), i.e. no memory outlives a call.
inline std::mutex &pool_mutex() {
    static std::mutex mu;
    return mu;
}
inline cudaMemPool_t *pool_table() {
    static cudaMemPool_t pools[64] = {};
    return pools;
}
inline cudaMemPool_t lib_pool(int dev) {
    cudaMemPool_t *pools = pool_table();
    if (dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(pool_mutex());
    if (!pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&pools[dev], &props) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
        } else {
            pools[dev] = nullptr;
            cudaGetLastError();
        }
    }
    return pools[dev];
}
// caching on: release threshold = max (keep everything); off: threshold 0 and trim now
inline bool set_pool_caching(int dev, bool on) {
    cudaMemPool_t pool = lib_pool(dev);
    if (!pool) return false;
    uint64_t thr = on ? UINT64_MAX : 0;
    if (cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr) != cudaSuccess) return false;
    return on || cudaMemPoolTrimTo(pool, 0) == cudaSuccess;
}

inline cudaError_t lib_malloc_async(void **p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidDevice;
    cudaMemPool_t pool = lib_pool(dev);
    if (!pool) return cudaMallocAsync(p, bytes, s);
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

// Compiled shape menus of the FP32 and complex translation units for a given b8 (autotuning):
// writes up to `max` shapes as {D, CW, tiles_per_warp, groups_per_step}, returns the count.
int f32_shape_menu(int b8, int (*out)[4], int max);
int c64_shape_menu(int b8, int (*out)[4], int max);

}  // namespace elpa_b200_host
