// Throughput microbenchmark of tcgen05.mma forms used by k_fused3 (tools only, not product).
// mode 0: cta_group::2 SS M=256 N=256 K=16 (bf16); 1: cta_group::2 TS (A in TMEM);
// mode 2: cta_group::2 SS N=128; mode 3: cta_group::1 SS M=128 N=256.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_1907_12933_b200/csrc/tc_ptx.cuh"
using namespace mlpv::tc;

__device__ __forceinline__ void mma1_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) { mma_f16_ss(d, a, b, idesc, acc); }

__device__ unsigned int g_sink;
__device__ uint4 g_src[2048];                       // 32 KB bulk-copy source (L2-resident)
__device__ uint4 g_src2[1 << 19];                   // 8 MB bulk-copy source (mode 35)
template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(768) k_bench(int reps, unsigned long long* cyc) {
  constexpr bool ONE = MODE == 3 || MODE == 31 || MODE == 32 || MODE == 33 || MODE == 34 || MODE == 35;   // cta_group::1 M128 N256 (N16 for 31)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t ready, done, scratch[4], pre;
  __shared__ uint32_t tbase;
  const uint32_t rank = cluster_ctarank();
  const int t = threadIdx.x, w = t >> 5;
  uint8_t* sA = smem;                 // 4 x 16 KB
  uint8_t* sB = smem + 4 * 16384;     // 4 x 16 KB
  for (int i = t; i < 8 * 16384 / 16; i += blockDim.x) {
    if (MODE == 20) {                                  // A: fp16 subnormal levels 0..15, B: random fp16 |x| < 0.125
      uint32_t x = (uint32_t)(i * 2654435761u) ^ (rank * 97u) ^ 0x9e3779b9u;
      uint32_t v[4];
      for (int k = 0; k < 4; k++) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        if (i < 4 * 16384 / 16) v[k] = (x & 0xFu) | (((x >> 8) & 0xFu) << 16);
        else v[k] = (0x2c00u | (x & 0x3ffu) | ((x >> 2) & 0x8000u)) | ((0x2c00u | ((x >> 16) & 0x3ffu) | ((x << 14) & 0x80000000u)) & 0xffff0000u) ;
      }
      reinterpret_cast<uint4*>(smem)[i] = make_uint4(v[0], v[1], v[2], v[3]);
    } else if (MODE >= 7) {                            // random bf16 in [-1, 1) / [0, 1)
      uint32_t x = (uint32_t)(i * 2654435761u) ^ (rank * 97u);
      uint32_t v[4];
      for (int k = 0; k < 4; k++) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        const uint32_t lo = 0x3f00u | (x & 0x7fu) | ((x >> 8) & 0x8000u), hi = 0x3e80u | ((x >> 16) & 0x7fu);
        v[k] = lo | (hi << 16);
      }
      reinterpret_cast<uint4*>(smem)[i] = make_uint4(v[0], v[1], v[2], v[3]);
    } else reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  }
  if (t == 0) {
    mbar_init(&ready, (!ONE && rank == 0) ? 2 : 1); mbar_init(&done, 1);
    for (int i = 0; i < 4; i++) mbar_init(&scratch[i], 1);
    mbar_init(&pre, 1);
    fence_mbar_init();
  }
  if (w == 0) { if (ONE) { tmem_alloc(&tbase, 512); tmem_relinquish(); } else { tmem_alloc2(&tbase, 512); tmem_relinquish2(); } }
  fence_proxy_async();
  fence_before();
  cluster_sync();
  fence_after();
  const uint32_t tb = tbase;
  if (t == 0) { if (rank == 0 || ONE) mbar_arrive(&ready); else mbar_arrive_cluster(&ready, 0); }
  if (t == 0) mbar_arrive(&pre);                       // phase 0 of `pre` completes: waits on it are no-ops
  const bool issuer = (ONE) ? (t == 0) : (rank == 0 && t == 0 && MODE != 15 && MODE != 25 && MODE != 27);
  __shared__ volatile int stop;
  if (t == 0) stop = 0;
  __syncthreads();
  __shared__ unsigned long long ld_cnt;
  if (t == 0) ld_cnt = 0;
  __syncthreads();
  if (MODE == 19 && w == 4 && rank == 0) {
    // second issuer: small TS MMAs (N = 16, A from TMEM cols 256.., D cols 496..) like layer 3
    const bool el = elect_one();
    unsigned long long n = 0;
    const uint32_t id3 = idesc_f16(256, 16, 0, 0);
    const uint64_t bd = sdesc_sw128(smem_u32(smem + 8 * 16384));
    while (!stop) {
      if (el) {
#pragma unroll
        for (int g = 0; g < 8; g++) mma2_f16_ts(tbase + 496, tbase + 256 + 16 * g, bd, id3, g ? 1u : 0u);
      }
      __syncwarp();
      n++;
      __nanosleep(400);
    }
    if (el && blockIdx.x == 0) printf("  L3-like batches issued: %llu\n", n);
  } else if ((MODE == 24 || MODE == 25 || MODE == 26 || MODE == 27 || MODE == 28) && w >= 4 && w < 12) {
    // epilogue-like: 8 warps (two per lane quadrant), per 16-column group: prefetch ld16 of the next
    // group, ~40 ALU ops, st16 in place, wait::ld
    const uint32_t loff = (uint32_t)(32 * (w & 3)) << 16;
    const uint32_t cb = 256u + 128u * (uint32_t)((w - 4) >> 2);
    unsigned long long n = 0;
    uint32_t buf[2][16];
    long long tst = 0, tld = 0;
    tmem_ld16(tbase + loff + cb, buf[0]);
    tmem_ld_wait();
    const long long t0 = clock64();
    while (!stop) {
#pragma unroll 2
      for (int g = 0; g < 8; g++) {
        uint32_t (&v)[16] = buf[g & 1];
        tmem_ld16(tbase + loff + cb + 16 * ((g + 1) & 7), buf[(g + 1) & 1]);
        uint32_t hl[16];
#pragma unroll
        for (int k = 0; k < 16; k++) hl[k] = (v[k] * 2654435761u) ^ (v[(k + 3) & 15] >> 3);
        const long long a0 = clock64();
        tmem_st16(tbase + loff + cb + 16 * g, hl);
        if (MODE == 26 || MODE == 27 || MODE == 28) tmem_st_wait();
        const long long a1 = clock64();
        tmem_ld_wait();
        const long long a2 = clock64();
        tst += a1 - a0; tld += a2 - a1;
      }
      tmem_st_wait();
      n += 8;
      if ((MODE == 25 || MODE == 27) && n >= 8 * 4000) break;
    }
    const long long t1 = clock64();
    if ((t & 31) == 0 && (w == 4 || w == 7) && (blockIdx.x == 0 || blockIdx.x == 1))
      printf("  w%d: %.1f cycles per group, st16 issue %.1f, ld wait %.1f\n", w, (double)(t1 - t0) / n, (double)tst / n, (double)tld / n);
  } else if (MODE == 18 && w >= 4 && w < 8) {
    const uint32_t loff = (uint32_t)(32 * (w & 3)) << 16;
    unsigned long long n = 0;
    uint32_t v[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    const long long t0 = clock64();
    while (!stop) {
#pragma unroll
      for (int g = 0; g < 16; g++) {
        uint32_t x[16];
        tmem_ld16(tbase + loff + 256 + 16 * g, x);
        tmem_ld_wait();
        v[0] += x[3];
        tmem_st8(tbase + loff + 256 + 16 * g, v);
        tmem_st8(tbase + loff + 256 + 16 * g + 8, v);
      }
      tmem_st_wait();
      n += 16;
    }
    const long long t1 = clock64();
    if ((t & 31) == 0 && w == 4 && blockIdx.x == 0) printf("  ld16+2xst8 rate: %.1f cycles per group (warp)\n", (double)(t1 - t0) / n);
  } else if ((MODE == 14 || MODE == 15 || MODE == 16 || MODE == 17) && w >= 4 && w < 8) {
    const uint32_t loff = (uint32_t)(32 * (w & 3)) << 16;
    const uint32_t lcol = MODE == 16 ? 0u : (MODE == 17 ? 256u : 256u);
    unsigned long long n = 0;
    uint32_t acc = 0;
    const long long t0 = clock64();
    while (!stop) {
#pragma unroll
      for (int g = 0; g < 16; g++) {
        uint32_t v[16];
        tmem_ld16(tbase + loff + lcol + 16 * g, v);
        tmem_ld_wait();
        acc += v[0] ^ v[15];
      }
      n += 16;
      if (MODE == 15 && n >= 16 * 2000) break;
    }
    const long long t1 = clock64();
    if ((t & 31) == 0 && w == 4 && blockIdx.x == 0) printf("  ld16 rate: %.1f cycles per ld16+wait (warp), %.1f B/clk/SM (4 warps)\n",
        (double)(t1 - t0) / n, 4.0 * n * 32 * 16 * 4 / (double)(t1 - t0));
    if (acc == 0x1234567u) g_sink = acc;
  } else if (MODE == 35 && w == 12) {
    // background: a ring of 2 x 16 KB bulk copies in flight (from an 8 MB L2-resident source,
    // block-dependent offsets), into a 32 KB smem scratch
    __shared__ uint64_t rbar[2];
    uint8_t* scratch = smem + 8 * 16384;
    if (t == 384) { mbar_init(&rbar[0], 1); mbar_init(&rbar[1], 1); fence_mbar_init(); }
    __syncwarp();
    long long n = 0;
    const long long t0 = clock64();
    uint32_t ph[2] = {0, 0};
    const uint8_t* src = reinterpret_cast<const uint8_t*>(g_src2);
    if (t == 384)
      for (int i = 0; i < 2; i++) { mbar_expect_tx(&rbar[i], 16384); bulk_g2s(scratch + i * 16384, src + ((blockIdx.x * 7 + i) & 511) * 16384, 16384, &rbar[i]); }
    while (!stop) {
      const int i = (int)(n & 1);
      mbar_wait(&rbar[i], ph[i]);
      ph[i] ^= 1u;
      n++;
      if (t == 384) { mbar_expect_tx(&rbar[i], 16384); bulk_g2s(scratch + i * 16384, src + ((blockIdx.x * 7 + n + 1) & 511) * 16384, 16384, &rbar[i]); }
      __syncwarp();
    }
    for (int i = 0; i < 2; i++) mbar_wait(&rbar[(n + i) & 1], ph[(n + i) & 1]);
    const long long t1 = clock64();
    if (t == 384 && blockIdx.x == 0) printf("  2 x 16 KB ring beside the MMAs: %.1f B/clk/SM\n", 16384.0 * n / (double)(t1 - t0));
  } else if ((MODE == 33 || MODE == 34) && w == 12) {
    // background: bulk copies of 32 KB from global (L2) into a smem scratch, back to back
    __shared__ uint64_t cbar;
    uint8_t* scratch = smem + 8 * 16384;
    if (t == 384) { mbar_init(&cbar, 1); fence_mbar_init(); }
    __syncwarp();
    uint32_t ph = 0;
    long long n = 0;
    const long long t0 = clock64();
    while (!stop) {
      if (t == 384) {
        mbar_expect_tx(&cbar, 32768);
        bulk_g2s(scratch, reinterpret_cast<const uint8_t*>(g_src), 32768, &cbar);
      }
      __syncwarp();
      mbar_wait(&cbar, ph);
      ph ^= 1u;
      n++;
    }
    const long long t1 = clock64();
    if (t == 384 && blockIdx.x == 0) printf("  bulk g2s beside the MMAs: %.1f B/clk/SM\n", 32768.0 * n / (double)(t1 - t0));
  } else if ((w >= 4 && MODE >= 10 && MODE < 14) || (MODE == 28 && w >= 12) || ((MODE == 32 || MODE == 34) && w >= 4 && w < 12)) {
    // background load while the MMAs run (warps 4..11)
    uint32_t c0 = t, c1 = t * 7, c2 = t * 13, c3 = t * 31, acc = 0;
    uint8_t* scratch = smem + 8 * 16384;                 // 32 KB scratch
    int it = 0;
    while (!stop) {
      if (MODE == 10 || MODE == 12 || MODE == 28) {
#pragma unroll
        for (int r = 0; r < 10; r++) {
          const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
          const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
          c0 = hi1 ^ c1 ^ r; c1 = lo1; c2 = hi0 ^ c3 ^ (r * 3); c3 = lo0;
        }
        acc += c0 ^ c2;
      }
      if (MODE == 11 || MODE == 12 || MODE == 28 || MODE == 32 || MODE == 34) {
#pragma unroll
        for (int k = 0; k < 4; k++)
          *reinterpret_cast<uint4*>(scratch + ((t * 16 + (it * 4 + k) * 4096) & 32767)) = make_uint4(c0, c1, acc, it);
      }
      it++;
    }
    if (acc == 0x12345u) g_sink = acc;
  }
  if (issuer) {
    if (!ONE) mbar_wait_cluster(&ready, 0); else mbar_wait(&ready, 0);
    fence_after();
    const uint32_t N = MODE == 2 ? 128 : ((MODE == 29 || MODE == 31) ? 16 : (MODE == 30 ? 64 : 256));
    const uint32_t idesc = ONE ? idesc_f16(128, N, 1, 1) : (MODE == 20 ? idesc_f16(256, N, 0, 0) : idesc_f16(256, N, 1, 1));
    long long t0 = clock64();
    if (MODE == 21 || MODE == 22 || MODE == 23) {      // rings + per-stage readiness checks (k_fused3 issuer)
      uint32_t gsl = 0, wsl = 0;
      const bool el = true;
      for (int r = 0; r < reps / 4; r++)
        for (int kb = 0; kb < 13; kb++) {
          const uint32_t ab = smem_u32(smem + gsl * 16384), bb = smem_u32(smem + 6 * 16384 + wsl * 16384);
          if (++gsl == 6) gsl = 0;
          if (++wsl == 5) wsl = 0;
          const bool rdy = MODE == 21 ? (mbar_test(&pre, 0) & mbar_test(&pre, 0)) : true;
          mma2_f16_ss(tb, sdesc_sw128(ab), sdesc_sw128(bb), idesc, (kb | r) ? 1u : 0u);
          mma2_commit(&scratch[0], 0x3);
          mma2_commit(&scratch[1], 0x3);
          mma2_f16_ss(tb, sdesc_sw128(ab + 32u), sdesc_sw128(bb + 32u), idesc, 1u);
          if (MODE == 22) mbar_wait2(&pre, 0, &pre, 0);
          if (MODE == 23) { mbar_wait(&pre, 0); mbar_wait(&pre, 0); }
          mma2_f16_ss(tb, sdesc_sw128(ab + 64u), sdesc_sw128(bb + 64u), idesc, 1u);
          mma2_f16_ss(tb, sdesc_sw128(ab + 96u), sdesc_sw128(bb + 96u), idesc, 1u);
          if (MODE == 21 && !rdy) mbar_wait2(&pre, 0, &pre, 0);
        }
    } else if (MODE == 13) {                             // k_fused3's rings: A 6 x 16 KB, B 5 x 16 KB
      uint32_t gsl = 0, wsl = 0;
      for (int r = 0; r < reps / 4; r++)
        for (int kb = 0; kb < 13; kb++) {
          const uint32_t ab = smem_u32(smem + gsl * 16384), bb = smem_u32(smem + 6 * 16384 + wsl * 16384);
          if (++gsl == 6) gsl = 0;
          if (++wsl == 5) wsl = 0;
          const int nk = kb == 12 ? 2 : 4;
#pragma unroll
          for (int kk = 0; kk < 4; kk++)
            if (kk < nk) mma2_f16_ss(tb, sdesc_sw128(ab + 32u * kk), sdesc_sw128(bb + 32u * kk), idesc, (kb | kk) ? 1u : 0u);
          mma2_commit(&scratch[0], 0x3);
          mma2_commit(&scratch[1], 0x3);
        }
    } else
    for (int r = 0; r < reps; r++)
      for (int kb = 0; kb < 4; kb++) {
        if (MODE == 5 || MODE == 6) { mbar_wait(&pre, 0); mbar_wait(&pre, 0); fence_after(); }
#pragma unroll
        for (int kk = 0; kk < 4; kk++) {
          const uint64_t ad = sdesc_sw128(smem_u32(sA + kb * 16384 + kk * 32));
          const uint64_t bd = sdesc_sw128(smem_u32(sB + kb * 16384 + kk * 32));
          const uint32_t acc = (r | kb | kk) ? 1u : 0u;
          if (MODE == 0 || MODE == 2 || (MODE >= 4 && MODE < 16) || MODE == 18 || MODE == 19 || MODE == 20 || MODE == 24 || MODE == 26 || MODE == 28 || MODE == 29 || MODE == 30) mma2_f16_ss(tb, ad, bd, idesc, acc);
          else if (MODE == 1) mma2_f16_ts(tb, tb + 256 + kb * 32 + kk * 8, bd, idesc, acc);
          else if (MODE == 16 || MODE == 17) mma2_f16_ts(tb + 256, tb + kb * 32 + kk * 8, bd, idesc_f16(256, 128, 1, 1), acc);
          else mma1_ss(tb, ad, bd, idesc, acc);
        }
        if (MODE == 4 || MODE == 6) { mma2_commit(&scratch[0], 0x3); mma2_commit(&scratch[1], 0x3); }
      }
    if (ONE) mma_commit(&done); else mma2_commit(&done, 0x3);
    mbar_wait(&done, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = (unsigned long long)(t1 - t0);
  }
  if (t == 0) {                                        // stop the background warps of both CTAs
    if (issuer || ONE) stop = 1;
  }
  if (!ONE) { if (t < 32 && !issuer) {} }
  __syncwarp();
  if (!issuer && t == 0 && !ONE && MODE != 15 && MODE != 25 && MODE != 27) { mbar_wait(&done, 0); stop = 1; }
  fence_before();
  __syncthreads();
  cluster_sync();
  fence_after();
  if (w == 0) { if (ONE) tmem_dealloc(tb, 512); else tmem_dealloc2(tb, 512); }
}

template <int MODE>
void run(const char* name) {
  constexpr bool ONE = MODE == 3 || MODE == 31 || MODE == 32 || MODE == 33 || MODE == 34 || MODE == 35;
  const size_t smem = (MODE == 13 || MODE >= 21 ? 13 : 10) * 16384 + 1024;
  cudaFuncSetAttribute(k_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  const int reps = 2000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int nt = (MODE == 28 || MODE >= 32) ? 768 : (MODE >= 10 ? 384 : 128);
  k_bench<MODE><<<148, nt, smem>>>(10, cyc);
  cudaEventRecord(e0);
  k_bench<MODE><<<148, nt, smem>>>(reps, cyc);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double M = ONE ? 128 : 256, N = MODE == 2 ? 128 : ((MODE == 29 || MODE == 31) ? 16 : (MODE == 30 ? 64 : 256));
  const double groups = ONE ? 148 : 74;
  const double flops = (MODE == 13 || (MODE >= 21 && MODE < 29)) ? 2.0 * M * N * 16 * 52 * (reps / 4) * groups : MODE == 13 ? 2.0 * M * N * 16 * 50 * (reps / 4) * groups : 2.0 * M * N * 16 * 16 * reps * groups;
  printf("%-28s err=%d  %.3f ms  %.1f TFLOP/s  cycles/MMA (cluster 0) %.1f\n", name, (int)e, ms, flops / (ms * 1e-3) / 1e12,
         (double)c / ((MODE >= 21 && MODE < 29) ? 52.0 * (reps / 4) : MODE == 13 ? 50.0 * (reps / 4) : 16.0 * reps));
}

int main() {
  run<0>("2CTA SS M256 N256 K16");
  run<3>("1CTA SS M128 N256 K16");
  run<29>("2CTA SS M256 N16 K16");
  run<30>("2CTA SS M256 N64 K16");
  run<31>("1CTA SS M128 N16 K16");
  run<32>("1CTA M128 N256 + 8w STS");
  run<33>("1CTA M128 N256 + bulk g2s");
  run<34>("1CTA M128 N256 + STS + bulk");
  run<35>("1CTA M128 N256 + 2x16KB ring");
  return 0;
}
