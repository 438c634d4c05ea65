// Test-only: cuRAND's device Philox4x32-10 (curand_philox4x32_x.h) as a library pin for the
// oracle's Philox (reading C15).  Not part of the product library.
#include <cuda_runtime.h>
#include <curand_kernel.h>

__global__ void k_ref(const uint4* ctr, const uint2* key, uint4* out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = curand_Philox4x32_10(ctr[i], key[i]);
}

extern "C" int curand_philox_ref(const void* ctr, const void* key, void* out, int n) {
  k_ref<<<(n + 255) / 256, 256>>>(static_cast<const uint4*>(ctr), static_cast<const uint2*>(key),
                                   static_cast<uint4*>(out), n);
  return (int)cudaDeviceSynchronize();
}
