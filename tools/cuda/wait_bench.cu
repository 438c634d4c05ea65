// How long do mbarrier.try_wait (with / without a suspend-time hint) and __nanosleep take on a barrier
// that does not complete?  (tools only)
#include <cstdio>
#include <cstdint>
#include "../../paper_1907_12933_b200/csrc/tc_ptx.cuh"
using namespace mlpv::tc;

__device__ __forceinline__ bool try_nohint(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(phase) : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool test_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(phase) : "memory");
  return ok != 0;
}
__global__ void k(int mode, unsigned long long* out) {
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  const int n = 200;
  int hits = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    bool ok;
    if (mode == 0) ok = mbar_try(&bar, 0);            // hint 20000 ns
    else if (mode == 1) ok = try_nohint(&bar, 0);
    else if (mode == 2) ok = test_wait(&bar, 0);
    else { __nanosleep(mode); ok = false; }
    hits += ok;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / n; out[1] = hits; }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  int modes[] = {0, 1, 2, 32, 128, 512, 2000};
  for (int m : modes) {
    k<<<1, 32>>>(m, d);
    unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("mode %5d: %llu cycles per call (hits %llu)\n", m, h[0], h[1]);
  }
  return 0;
}
