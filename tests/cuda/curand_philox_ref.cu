// Test-only reference (not product code): cuRAND's own Philox4x32-10 (curand_philox4x32_x.h) on the
// device, for tests/test_gpu_rng_curand.py.  out[i] = curand_Philox4x32_10(ctr[i], key[i]).
#include <cstdint>
#include <cuda_runtime.h>
#include <curand_philox4x32_x.h>

__global__ void ref_kernel(const uint4* ctr, const uint2* key, uint4* out, unsigned long long n) {
    const unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = curand_Philox4x32_10(ctr[i], key[i]);
}

extern "C" int curand_philox_ref(const void* ctr, const void* key, void* out, unsigned long long n, void* stream) {
    if (n == 0) return 0;
    ref_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        (const uint4*)ctr, (const uint2*)key, (uint4*)out, n);
    return (int)cudaGetLastError();
}
