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
#include "../../paper_1907_12933_b200/csrc/tc_ptx.cuh"
using namespace mlpv::tc;

constexpr int kStages = 4;
constexpr uint32_t kStage = 16384;

__global__ void __launch_bounds__(128) k_bulk(const uint8_t* buf, size_t bytes, int passes, unsigned long long* sink) {
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
    const size_t off = (size_t)blockIdx.x * 37 % n;
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
  const int smem = kStages * kStage + 1024;
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // bulk copies, every SM streaming the same L2-resident buffer (the weight-streaming pattern)
  for (size_t B : {(size_t)1 << 20, (size_t)6 << 20, (size_t)16 << 20}) {
    const int passes = (int)((size_t)(256u << 20) / B);
    k_bulk<<<sms, 128, smem>>>(buf, B, 1, sink);                       // warm
    cudaEventRecord(e0);
    k_bulk<<<sms, 128, smem>>>(buf, B, passes, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tot = (double)B * passes * sms;
    printf("{\"test\": \"bulk_same_buffer\", \"buffer_MB\": %.0f, \"GB_per_s\": %.1f, \"B_per_clk_per_SM_at_max_clk\": %.1f, \"ms\": %.3f}\n",
           B / 1048576.0, tot / ms / 1e6, tot / (ms * 1e-3) / sms / (clk * 1e3), ms);
  }
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
