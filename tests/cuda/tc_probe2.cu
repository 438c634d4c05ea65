// Test-only probe of the 2-CTA (cta_group::2) tcgen05 primitives in tc_ptx.cuh: a cluster of two
// CTAs computes D[256 x N] = A[256 x K] * B[N x K]^T; CTA r holds A rows [128r, 128r+128) and B rows
// [rN/2, (r+1)N/2) at identical shared-memory offsets; the leader issues tcgen05.mma.cta_group::2
// and commits to both CTAs' barriers; each CTA reads its own 128 accumulator rows from its TMEM.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../paper_1907_12933_b200/csrc/tc_ptx.cuh"

using namespace mlpv::tc;

// mode: 0 bf16 SS, 1 bf16 TS (A in TMEM)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128)
    k_probe2(int mode, const uint8_t* A, const uint8_t* B, uint32_t* D, int N, int K) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t ready, done;
  __shared__ uint32_t tbase;
  const uint32_t rank = cluster_ctarank();
  const int row_bytes = K * 2, nkb = row_bytes / 128, nh = N / 2;
  uint8_t* sA = smem;
  uint8_t* sB = smem + 128 * row_bytes;
  const int t = threadIdx.x, w = t >> 5;
  if (t == 0) {
    mbar_init(&ready, rank == 0 ? 2 : 1);
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (w == 0) { tmem_alloc2(&tbase, 512); tmem_relinquish2(); }
  fence_before();
  cluster_sync();
  fence_after();
  const uint32_t tb = tbase;
  const uint8_t* Ar = A + (size_t)rank * 128 * row_bytes;
  const uint8_t* Br = B + (size_t)rank * nh * row_bytes;
  for (int e = t; e < 128 * row_bytes / 16; e += 128) {
    const int r = e / (row_bytes / 16), c = e % (row_bytes / 16);
    *reinterpret_cast<uint4*>(sA + (c / 8) * 128 * 128 + sw128_off(r, (c % 8) * 16)) =
        *reinterpret_cast<const uint4*>(Ar + (size_t)r * row_bytes + c * 16);
  }
  for (int e = t; e < nh * row_bytes / 16; e += 128) {
    const int r = e / (row_bytes / 16), c = e % (row_bytes / 16);
    *reinterpret_cast<uint4*>(sB + (c / 8) * nh * 128 + sw128_off(r, (c % 8) * 16)) =
        *reinterpret_cast<const uint4*>(Br + (size_t)r * row_bytes + c * 16);
  }
  const uint32_t a_col = 256;
  if (mode == 1) {
    for (int c0 = 0; c0 < row_bytes / 4; c0 += 8) {
      uint32_t v[8];
      for (int i = 0; i < 8; i++) v[i] = *reinterpret_cast<const uint32_t*>(Ar + (size_t)t * row_bytes + 4 * (c0 + i));
      tmem_st8(tb + ((uint32_t)(w * 32) << 16) + a_col + c0, v);
    }
    tmem_st_wait();
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  if (t == 0) {
    if (rank == 0) mbar_arrive(&ready);
    else mbar_arrive_cluster(&ready, 0);
  }
  if (rank == 0 && t == 0) {
    mbar_wait_cluster(&ready, 0);
    fence_after();
    const uint32_t idesc = idesc_f16(256, N, 1, 1);
    int step = 0;
    for (int kb = 0; kb < nkb; kb++)
      for (int kk = 0; kk < 4; kk++) {
        const uint64_t bd = sdesc_sw128(smem_u32(sB + kb * nh * 128 + kk * 32));
        if (mode == 0) mma2_f16_ss(tb, sdesc_sw128(smem_u32(sA + kb * 128 * 128 + kk * 32)), bd, idesc, step > 0);
        else mma2_f16_ts(tb, tb + a_col + kb * 32 + kk * 8, bd, idesc, step > 0);
        step++;
      }
    mma2_commit(&done, 0x3);
  }
  __syncwarp();
  mbar_wait(&done, 0);
  fence_after();
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tb + ((uint32_t)(w * 32) << 16) + c0, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; i++)
      if (c0 + i < N) D[(size_t)(128 * rank + t) * N + c0 + i] = r[i];
  }
  fence_before();
  cluster_sync();
  fence_after();
  if (w == 0) tmem_dealloc2(tb, 512);
}

extern "C" int tc_probe2(int mode, const void* A, const void* B, void* D, int N, int K) {
  const size_t smem = (size_t)(128 + N / 2) * K * 2 + 1024;
  cudaFuncSetAttribute(k_probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_probe2<<<2, 128, smem>>>(mode, static_cast<const uint8_t*>(A), static_cast<const uint8_t*>(B),
                             static_cast<uint32_t*>(D), N, K);
  return (int)cudaDeviceSynchronize();
}
