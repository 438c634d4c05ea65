// Test-only probe of the tcgen05 building blocks in paper_1907_12933_b200/csrc/tc_ptx.cuh:
// one CTA computes D[128 x N] = A[128 x K] * B[N x K]^T with the operands staged exactly as the
// product kernel stages them (SWIZZLE_128B K-major smem tiles, or A written to TMEM for the TS
// form).  Compared against torch.matmul by tests/test_tcgen05_gpu.py.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../paper_1907_12933_b200/csrc/tc_ptx.cuh"

using namespace mlpv::tc;

// mode: 0 bf16 SS, 1 f16 SS, 2 f16 TS, 3 bf16 TS, 4 u8*s8 SS, 5 u8*s8 TS
__global__ void __launch_bounds__(128) k_probe(int mode, const uint8_t* A, const uint8_t* B, uint32_t* D, int N, int K) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // SW128 needs 1 KiB alignment
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int esz = mode >= 4 ? 1 : 2;
  const int row_bytes = K * esz;                  // bytes of K per row
  const int nkb = row_bytes / 128;                // 128-byte K blocks
  uint8_t* sA = smem;
  uint8_t* sB = smem + 128 * row_bytes;
  const int t = threadIdx.x, w = t >> 5;
  if (w == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  // stage A and B (SW128 K-major, K blocks of 128 bytes stored tile after tile)
  for (int e = t; e < 128 * row_bytes / 16; e += 128) {
    const int r = e / (row_bytes / 16), c = e % (row_bytes / 16);
    const int kb = c / 8, ch = c % 8;
    *reinterpret_cast<uint4*>(sA + kb * 128 * 128 + sw128_off(r, ch * 16)) =
        *reinterpret_cast<const uint4*>(A + (size_t)r * row_bytes + c * 16);
  }
  for (int e = t; e < N * row_bytes / 16; e += 128) {
    const int r = e / (row_bytes / 16), c = e % (row_bytes / 16);
    const int kb = c / 8, ch = c % 8;
    *reinterpret_cast<uint4*>(sB + kb * N * 128 + sw128_off(r, ch * 16)) =
        *reinterpret_cast<const uint4*>(B + (size_t)r * row_bytes + c * 16);
  }
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = tbase;
  const uint32_t a_col = 256;                     // TS: A lives in columns 256.. (32-bit cells)
  const bool ts = mode == 2 || mode == 3 || mode == 5;
  if (ts) {
    // row m = lane m = thread m; column a_col + c holds bytes [4c, 4c+4) of the row
    for (int c0 = 0; c0 < row_bytes / 4; c0 += 8) {
      uint32_t v[8];
      for (int i = 0; i < 8; i++) v[i] = *reinterpret_cast<const uint32_t*>(A + (size_t)t * row_bytes + 4 * (c0 + i));
      tmem_st8(tb + ((uint32_t)(w * 32) << 16) + a_col + c0, v);
    }
    tmem_st_wait();
    fence_before();
    __syncthreads();
    fence_after();
  }
  if (t == 0) {
    uint32_t idesc;
    if (mode == 0 || mode == 3) idesc = idesc_f16(128, N, 1, 1);
    else if (mode == 1 || mode == 2) idesc = idesc_f16(128, N, 0, 0);
    else idesc = idesc_i8(128, N, 0, 1);
    int step = 0;
    for (int kb = 0; kb < nkb; kb++) {
      for (int kk = 0; kk < 4; kk++) {            // 32 bytes of K per instruction
        const uint64_t bd = sdesc_sw128(smem_u32(sB + kb * N * 128 + kk * 32));
        const uint32_t acc = step > 0 ? 1u : 0u;
        if (!ts) {
          const uint64_t ad = sdesc_sw128(smem_u32(sA + kb * 128 * 128 + kk * 32));
          if (mode >= 4) mma_i8_ss(tb, ad, bd, idesc, acc); else mma_f16_ss(tb, ad, bd, idesc, acc);
        } else {
          const uint32_t at = tb + a_col + (uint32_t)(kb * 32 + kk * 8);
          if (mode >= 4) mma_i8_ts(tb, at, bd, idesc, acc); else mma_f16_ts(tb, at, bd, idesc, acc);
        }
        step++;
      }
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  fence_after();
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tb + ((uint32_t)(w * 32) << 16) + c0, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; i++) if (c0 + i < N) D[(size_t)t * N + c0 + i] = r[i];
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (w == 0) tmem_dealloc(tb, 512);
}

extern "C" int tc_probe(int mode, const void* A, const void* B, void* D, int N, int K) {
  const int esz = mode >= 4 ? 1 : 2;
  const size_t smem = (size_t)(128 + N) * K * esz + 1024;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_probe<<<1, 128, smem>>>(mode, static_cast<const uint8_t*>(A), static_cast<const uint8_t*>(B),
                            static_cast<uint32_t*>(D), N, K);
  return (int)cudaDeviceSynchronize();
}
