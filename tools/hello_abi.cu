// Interop check: a statically-linked-cudart .so launched on torch's stream.
#include <cuda_runtime.h>
__global__ void inc(double* p, long n) { long i = blockIdx.x * (long)blockDim.x + threadIdx.x; if (i < n) p[i] += 1.0; }
extern "C" int hello_inc(double* p, long n, void* stream) {
  inc<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(p, n);
  return (int)cudaGetLastError();
}
