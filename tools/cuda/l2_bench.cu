// L2 -> SM bandwidth and L2 capacity on the B200 (tools only, not product; SURVEY.md §8(d) asks for
// both before the large configs' weight streaming is judged).
//  bulk: every CTA (one per SM) streams a buffer of B bytes (all CTAs read the same buffer, as
//        k_large / k_fused3 stream the same weight tiles) with cp.async.bulk into a 4-stage smem ring
//        of 16 KB stages, one issuing thread, mbarrier complete_tx -- the producer pattern of the
//        kernels.  Reported: bytes delivered to shared memory per second, whole GPU.
//  ldg:  every thread reads its slice of a buffer of B bytes with 16-byte loads, the grid covering
//        the buffer once per pass (each byte read once per pass); passes repeat.  B below the L2
//        capacity: L2 bandwidth; above it: HBM bandwidth -- the knee is the usable L2 capacity.
// usage: l2_bench            (prints one JSON line per measurement)
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <type_traits>
#include "../../paper_1907_12933_b200/csrc/tc_ptx.cuh"
using namespace mlpv::tc;

constexpr uint32_t kStage = 16384;

template <int kStages>
__global__ void __launch_bounds__(128) k_bulk(const uint8_t* buf, size_t bytes, int passes, unsigned long long* sink, int stagger) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[kStages];
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; i++) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const size_t n = bytes / kStage;
    // stagger the start so that the CTAs do not all read the same line at the same time
    const size_t off = stagger ? (size_t)blockIdx.x * 37 % n : 0;
    uint64_t it = 0;
    for (int p = 0; p < passes; p++)
      for (size_t i = 0; i < n; i++, it++) {
        const uint32_t st = it % kStages, ph = (it / kStages) & 1u;
        if (it >= kStages) mbar_wait(&full[st], ph ^ 1u);          // stage consumed (previous phase)
        mbar_expect_tx(&full[st], kStage);
        bulk_g2s(sm + st * kStage, buf + ((i + off) % n) * kStage, kStage, &full[st]);
      }
    for (uint64_t j = it > kStages ? it - kStages : 0; j < it; j++) mbar_wait(&full[j % kStages], (j / kStages) & 1u);
    sink[blockIdx.x] = *reinterpret_cast<volatile unsigned long long*>(sm);
  }
}


// multicast variant: clusters of C CTAs; stage s is fetched once, by CTA s % C, and multicast into the
// same slot of every CTA of the cluster (cp.async.bulk ... .multicast::cluster); each CTA waits for its
// full barrier and then arrives on the issuing CTA's empty barrier (C arrivals free the slot).
template <int C, int S>
__global__ void __launch_bounds__(128) k_bulk_mc(const uint8_t* buf, size_t bytes, int passes, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[S], empty[S];
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], C); }
    fence_mbar_init();
  }
  __syncthreads();
  cluster_sync();
  if (threadIdx.x == 0) {
    const size_t n = bytes / kStage;
    const uint16_t mask = (uint16_t)((1u << C) - 1u);
    // S - 1 stages in flight: stage `it` is armed / issued, stage it - (S - 1) is consumed
    const uint64_t N = (uint64_t)passes * n;
    for (uint64_t it = 0; it < N + S - 1; it++) {
      if (it < N) {
        const uint32_t st = it % S, ph = (it / S) & 1u;
        mbar_expect_tx(&full[st], kStage);
        if (it % C == rank) {
          if (it >= S) mbar_wait(&empty[st], ph ^ 1u);          // every CTA has consumed the slot
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
              ::"r"(smem_u32(sm + st * kStage)), "l"(buf + (it % n) * kStage), "r"(kStage), "r"(smem_u32(&full[st])), "h"(mask)
              : "memory");
        }
      }
      if (it >= (uint64_t)(S - 1)) {
        const uint64_t j = it - (S - 1);
        mbar_wait(&full[j % S], (j / S) & 1u);
        mbar_arrive_cluster(&empty[j % S], (uint32_t)(j % C));
      }
    }
    sink[blockIdx.x] = *reinterpret_cast<volatile unsigned long long*>(sm);
  }
  __syncthreads();
  cluster_sync();
}

__global__ void __launch_bounds__(512) k_ldg(const uint4* buf, size_t n16, int passes, unsigned long long* sink) {
  uint32_t x = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int p = 0; p < passes; p++)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += 4 * stride) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; u++) v[u] = i + u * stride < n16 ? __ldcg(buf + i + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < 4; u++) x ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
  if (x == 0x12345678u) sink[0] = x;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  printf("{\"device_sms\": %d, \"l2_bytes_attr\": %d}\n", sms, l2);
  const size_t maxB = (size_t)1 << 30;
  uint8_t* buf;
  cudaMalloc(&buf, maxB);
  cudaMemset(buf, 1, maxB);
  unsigned long long* sink;
  cudaMalloc(&sink, 4096 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto bulk = [&](auto stc) {
    constexpr int kS = decltype(stc)::value;
    const int smem = kS * kStage + 1024;
    cudaFuncSetAttribute(k_bulk<kS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int stagger = 1; stagger >= 0; stagger--)
      for (size_t B : {(size_t)1 << 20, (size_t)6 << 20}) {
        const int passes = (int)((size_t)(256u << 20) / B);
        k_bulk<kS><<<sms, 128, smem>>>(buf, B, 1, sink, stagger);              // warm
        cudaEventRecord(e0);
        k_bulk<kS><<<sms, 128, smem>>>(buf, B, passes, sink, stagger);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double tot = (double)B * passes * sms;
        printf("{\"test\": \"bulk_same_buffer\", \"stages_16KB\": %d, \"stagger\": %d, \"buffer_MB\": %.0f, \"GB_per_s\": %.1f, "
               "\"B_per_clk_per_SM_at_max_clk\": %.1f, \"ms\": %.3f}\n",
               kS, stagger, B / 1048576.0, tot / ms / 1e6, tot / (ms * 1e-3) / sms / (clk * 1e3), ms);
      }
  };
  // bulk copies, every SM streaming the same L2-resident buffer (the weight-streaming pattern);
  // stagger 0: every CTA walks the buffer in the same order from the same start (as the kernels do)
  bulk(std::integral_constant<int, 2>{});
  bulk(std::integral_constant<int, 4>{});
  bulk(std::integral_constant<int, 8>{});
  auto mc = [&](auto cc, auto sc) {
    constexpr int C = decltype(cc)::value, S = decltype(sc)::value;
    const int smem = S * kStage + 1024;
    cudaFuncSetAttribute(k_bulk_mc<C, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(sms / C * C));
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const size_t B = (size_t)6 << 20;
    const int passes = 40;
    cudaLaunchKernelEx(&cfg, k_bulk_mc<C, S>, (const uint8_t*)buf, B, 1, sink);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k_bulk_mc<C, S>, (const uint8_t*)buf, B, passes, sink);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tot = (double)B * passes * (sms / C * C);        // bytes delivered to shared memory
    printf("{\"test\": \"bulk_multicast\", \"cluster\": %d, \"stages_16KB\": %d, \"delivered_GB_per_s\": %.1f, "
           "\"delivered_B_per_clk_per_SM_at_max_clk\": %.1f, \"ms\": %.3f, \"err\": \"%s\"}\n",
           C, S, tot / ms / 1e6, tot / (ms * 1e-3) / (sms / C * C) / (clk * 1e3), ms, cudaGetErrorString(err));
  };
  mc(std::integral_constant<int, 2>{}, std::integral_constant<int, 4>{});
  mc(std::integral_constant<int, 2>{}, std::integral_constant<int, 8>{});
  mc(std::integral_constant<int, 4>{}, std::integral_constant<int, 8>{});
  // coalesced loads, each byte once per pass: the L2 capacity knee and the HBM bandwidth
  for (size_t mb : {8, 16, 32, 48, 64, 80, 96, 112, 128, 160, 192, 256, 512, 1024}) {
    const size_t B = mb << 20, n16 = B / 16;
    const int passes = (int)std::max<size_t>(2, (size_t)(8ull << 30) / B);
    k_ldg<<<sms * 4, 512>>>(reinterpret_cast<const uint4*>(buf), n16, 2, sink);   // warm (fills L2)
    cudaEventRecord(e0);
    k_ldg<<<sms * 4, 512>>>(reinterpret_cast<const uint4*>(buf), n16, passes, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tot = (double)B * passes;
    printf("{\"test\": \"ldg_sweep\", \"buffer_MB\": %zu, \"GB_per_s\": %.1f, \"ms\": %.3f}\n", mb, tot / ms / 1e6, ms);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
