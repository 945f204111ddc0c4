// host_common.h — host-side helpers shared by the library's translation units
// (elpa_b200.cu: FP64 path, elpa_b200_f32.cu: FP32 path).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

#include "../../include/elpa_b200.h"

namespace elpa_b200_host {

constexpr int kMaxSms = 148;

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
// CTA's critical path, but a next pass chained right behind waits for it.  Development
// override: ELPA_B200_PUB.
inline int pub_period() {
    static int v = [] {
        const char *e = getenv("ELPA_B200_PUB");
        int x = e ? atoi(e) : 32;
        return x >= 1 ? x : 32;
    }();
    return v;
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

}  // namespace elpa_b200_host
