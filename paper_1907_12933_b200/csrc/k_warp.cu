// k_warp.cu -- the enumerated-space kernel for small int8 nets (BASELINE config 3: 784-64-32-10,
// SUBSET spaces): one WARP per candidate at a time, its lanes the
// neurons, instead of k_small's one thread per candidate.
//
// k_small keeps a candidate's 64 + 32 + 10 potentials in one thread's registers (204 registers, 8
// warps per SM, latency-bound) and reads W2 from shared memory word by word (~600 issue slots per
// candidate, profiles/r2_cfg3_k_small_ncu.txt).  Here lane j owns layer-1 neurons j and j + 32,
// layer-2 neuron j and layer-3 neuron j; W2 / W3 rows live in the lanes' registers; the layer
// inputs are broadcast through 96 bytes of shared memory per warp (one byte store per neuron, four
// / two 16-byte loads); sign words are ballots; argmax, L-inf and the property are warp reductions.
//   layer 1 (a4)  the rank-|S| update of reading C14 / SURVEY a4: u1 = base + sum_k Delta[k][d_k]
//                 with the prefix over all digits but the last kept across the q consecutive
//                 candidates that share it (one table load pair per candidate);
//   layers 2, 3   DP4A (u8 x s8 -> s32), requant y = min(255, max(0, (acc + 2^(sh-1)) >> sh))
//                 (reading C18), exact;
//   a5, a7-a9     predicates on int32 potentials, covers of pairs (1,2) and (2,3) (C3-C8) OR-ed
//                 into the block's shared words, counts and the first counterexample per warp.
// Bit-exact against the oracle (tests/test_parity_gpu.py); eval / restriction / incremental runs
// stay on k_small.
#include <cuda_runtime.h>

#include <cstdint>

#include "mlpv_internal.cuh"

namespace mlpv {
namespace kw {

constexpr int kWarps = 8;
constexpr int kChunk = 64;                 // consecutive candidates per warp task

__device__ __forceinline__ int32_t dp4a_us(uint32_t a_u8x4, uint32_t b_s8x4, int32_t c) {
  int32_t d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a_u8x4), "r"(b_s8x4), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t iabs_u(int32_t d) { return (uint32_t)(d < 0 ? -d : d); }

struct Args {
  DevNet net;
  DevPert pert;
  DevProp prop;
  DevCov cov;
  DevResult res;
  BaseWS ws;
};

// FULL: n1 = 64, n2 = 32 (config 3's shape): every lane owns real neurons in layers 1 and 2, no
// per-lane predicates there
template <bool FULL>
__global__ void __launch_bounds__(32 * kWarps, 3) k_warp3(const __grid_constant__ Args a) {
  __shared__ uint32_t s_cov[256];
  __shared__ __align__(16) uint8_t s_h[kWarps][2][96];                // [warp][buffer] h1 (64) | h2 (32)
  __shared__ unsigned long long s_cnt[2], s_cex;
  const int b = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const DevNet& net = a.net;
  const int n1 = net.sizes[1], n2 = net.sizes[2], n3 = net.sizes[3];
  const int T = net.trace_len;
  const int sh1 = net.shift[0], sh2 = net.shift[1];
  const uint32_t nw = a.cov.n_words;
  for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x) s_cov[i] = 0;
  if (threadIdx.x < 2) s_cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_cex = kNone;

  // ---- per-lane constants: weight rows (s8x4 words), biases, base potentials and sign words
  uint32_t W2r[16], W3r[8];
  const int8_t* W2 = static_cast<const int8_t*>(net.W[1]);
  const int8_t* W3 = static_cast<const int8_t*>(net.W[2]);
#pragma unroll
  for (int m = 0; m < 16; m++) {
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 4; k++)
      if (lane < n2 && 4 * m + k < n1) v |= (uint32_t)(uint8_t)W2[lane * n1 + 4 * m + k] << (8 * k);
    W2r[m] = v;
  }
#pragma unroll
  for (int m = 0; m < 8; m++) {
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 4; k++)
      if (lane < n3 && 4 * m + k < n2) v |= (uint32_t)(uint8_t)W3[lane * n2 + 4 * m + k] << (8 * k);
    W3r[m] = v;
  }
  const int32_t b2 = lane < n2 ? static_cast<const int32_t*>(net.b[1])[lane] : 0;
  const int32_t b3 = lane < n3 ? static_cast<const int32_t*>(net.b[2])[lane] : 0;
  const int32_t* tr = static_cast<const int32_t*>(a.ws.trace) + (size_t)b * T;
  const bool in1a = FULL || lane < n1, in1b = FULL || lane + 32 < n1, in2 = FULL || lane < n2, in3 = lane < n3;
  const int32_t ub1a = in1a ? tr[net.loff[1] + lane] : 0, ub1b = in1b ? tr[net.loff[1] + lane + 32] : 0;
  const int32_t ub2 = in2 ? tr[net.loff[2] + lane] : 0, ub3 = in3 ? tr[net.loff[3] + lane] : 0;
  const uint32_t m1a = __ballot_sync(0xffffffffu, in1a), m1b = __ballot_sync(0xffffffffu, in1b);
  const uint32_t m2 = __ballot_sync(0xffffffffu, in2), m3 = __ballot_sync(0xffffffffu, in3);
  const uint32_t sb1a = __ballot_sync(0xffffffffu, ub1a >= 0) & m1a, sb1b = __ballot_sync(0xffffffffu, ub1b >= 0) & m1b;
  const uint32_t sb2 = __ballot_sync(0xffffffffu, ub2 >= 0) & m2, sb3 = __ballot_sync(0xffffffffu, ub3 >= 0) & m3;
  const int base_cls = a.ws.cls[b];
  int p12 = -1, p23 = -1;
  for (int p = 0; p < a.cov.n_pairs; p++) {
    if (a.cov.lower[p] == 1) p12 = p;
    if (a.cov.lower[p] == 2) p23 = p;
  }
  const int32_t tg2 = (int32_t)a.cov.tg_i[1], tg3 = (int32_t)a.cov.tg_i[2];
  const uint32_t th1 = (uint32_t)a.cov.th_i[0], th2 = (uint32_t)a.cov.th_i[1];
  const int K = a.pert.n_pixels, q = a.pert.n_levels;
  // the property, hoisted (kind 0: argmax unchanged, 1: target never, 2/3: the literal, C12)
  const int pkind = a.prop.kind, ptarget = a.prop.target;
  const int32_t pV = (int32_t)a.prop.V_i;
  const int pD = ptarget >= 0 ? ptarget : base_cls;
  const uint32_t pothers = m3 & ~(1u << (pD & 31));
  const int32_t r1 = sh1 > 0 ? (1 << (sh1 - 1)) : 0, r2 = sh2 > 0 ? (1 << (sh2 - 1)) : 0;
  const int32_t* delta = static_cast<const int32_t*>(a.ws.delta) + (size_t)b * K * q * n1;
  __syncthreads();

  const uint64_t begin = a.pert.begin, len = a.pert.end - a.pert.begin;
  const uint64_t nchunk = (len + kChunk - 1) / kChunk;
  unsigned long long my_chk = 0, my_v = 0, my_cex = kNone;
  int buf = 0;
  for (uint64_t ch = (uint64_t)blockIdx.x * kWarps + warp; ch < nchunk; ch += (uint64_t)gridDim.x * kWarps) {
    const uint64_t c0 = begin + ch * kChunk;
    const uint64_t c1 = c0 + kChunk < begin + len ? c0 + kChunk : begin + len;
    uint64_t hi = c0 / (uint64_t)q;                  // the digits above the last one, as a number
    int dl = (int)(c0 % (uint64_t)q);                // the last (least significant) digit
    int32_t pa = 0, pb = 0;                          // prefix: base + Delta of every digit but the last
    auto prefix = [&]() {
      pa = ub1a; pb = ub1b;
      uint64_t cc = hi;
      for (int k = K - 2; k >= 0; k--) {
        const int d = (int)(cc % (uint64_t)q);
        cc /= (uint64_t)q;
        const int32_t* row = delta + ((size_t)k * q + d) * n1;
        if (in1a) pa += __ldg(row + lane);
        if (in1b) pb += __ldg(row + lane + 32);
      }
    };
    prefix();
    const int32_t* last = delta + (size_t)(K - 1) * q * n1;   // rows of the last digit
    const int ncand = (int)(c1 - c0);
    for (int i = 0; i < ncand; i++) {
      // ---- layer 1: one table row for the last digit
      const int32_t* row = last + dl * n1;
      const int32_t u1a = in1a ? pa + __ldg(row + lane) : 0, u1b = in1b ? pb + __ldg(row + lane + 32) : 0;
      if (++dl == q) { dl = 0; hi++; if (i + 1 < ncand) prefix(); }
      const uint32_t sc1a = (__ballot_sync(0xffffffffu, u1a >= 0) & m1a) ^ sb1a;
      const uint32_t sc1b = (__ballot_sync(0xffffffffu, u1b >= 0) & m1b) ^ sb1b;
      const int nsc1 = __popc(sc1a) + __popc(sc1b);
      // ---- layer 2 (DP4A against the lane's W2 row; h1 broadcast through shared memory)
      uint8_t* hb = s_h[warp][buf];
      buf ^= 1;
      hb[lane] = (uint8_t)(in1a ? max(0, min(255, (u1a + r1) >> sh1)) : 0);      // requant, reading C18
      hb[32 + lane] = (uint8_t)(in1b ? max(0, min(255, (u1b + r1) >> sh1)) : 0);
      __syncwarp();
      const uint4* h4 = reinterpret_cast<const uint4*>(hb);
      int32_t acc2[4] = {b2, 0, 0, 0};                  // four independent DP4A chains
#pragma unroll
      for (int m4 = 0; m4 < 4; m4++) {
        const uint4 w = h4[m4];
        acc2[0] = dp4a_us(w.x, W2r[4 * m4], acc2[0]);
        acc2[1] = dp4a_us(w.y, W2r[4 * m4 + 1], acc2[1]);
        acc2[2] = dp4a_us(w.z, W2r[4 * m4 + 2], acc2[2]);
        acc2[3] = dp4a_us(w.w, W2r[4 * m4 + 3], acc2[3]);
      }
      int32_t u2 = (acc2[0] + acc2[1]) + (acc2[2] + acc2[3]);
      if (!in2) u2 = 0;
      const uint32_t sc2 = (__ballot_sync(0xffffffffu, u2 >= 0) & m2) ^ sb2;
      const int nsc2 = __popc(sc2);
      // ---- layer 3
      hb[64 + lane] = (uint8_t)(in2 ? max(0, min(255, (u2 + r2) >> sh2)) : 0);
      __syncwarp();
      int32_t acc3[4] = {b3, 0, 0, 0};
#pragma unroll
      for (int m4 = 0; m4 < 2; m4++) {
        const uint4 w = h4[4 + m4];
        acc3[0] = dp4a_us(w.x, W3r[4 * m4], acc3[0]);
        acc3[1] = dp4a_us(w.y, W3r[4 * m4 + 1], acc3[1]);
        acc3[2] = dp4a_us(w.z, W3r[4 * m4 + 2], acc3[2]);
        acc3[3] = dp4a_us(w.w, W3r[4 * m4 + 3], acc3[3]);
      }
      int32_t u3 = (acc3[0] + acc3[1]) + (acc3[2] + acc3[3]);
      if (!in3) u3 = 0;
      // ---- a7: argmax (lowest index on ties), property
      const int32_t top = __reduce_max_sync(0xffffffffu, in3 ? u3 : INT32_MIN);
      const int cls = __ffs(__ballot_sync(0xffffffffu, in3 && u3 == top)) - 1;
      bool viol;
      if (pkind == MLPV_PROP_THRESHOLD_LITERAL || pkind == MLPV_PROP_THRESHOLD_LITERAL_ALL) {
        const int32_t yD = __shfl_sync(0xffffffffu, u3, pD);
        const uint32_t gt = __ballot_sync(0xffffffffu, in3 && lane != pD && u3 > pV);
        viol = yD < pV && (pkind == MLPV_PROP_THRESHOLD_LITERAL_ALL ? gt == pothers : gt != 0);
      } else {
        viol = pkind == MLPV_PROP_TARGET_NEVER ? cls == ptarget : cls != base_cls;
      }
      if (viol) { my_v++; if (c0 + (uint64_t)i < my_cex) my_cex = c0 + (uint64_t)i; }
      // ---- a8: covers of pairs (1, 2) and (2, 3) (reading C3-C8), rare, warp-uniform branches
      if (p12 >= 0 && nsc1 <= 1) {
        bool cond = nsc1 == 1;
        if (!cond) {
          const uint32_t d = max(in1a ? iabs_u(u1a - ub1a) : 0u, in1b ? iabs_u(u1b - ub1b) : 0u);
          cond = __reduce_max_sync(0xffffffffu, d) >= th1;
        }
        if (cond) {
          const uint32_t vc2 = __ballot_sync(0xffffffffu, in2 && iabs_u(u2 - ub2) >= (uint32_t)tg2) & ~sc2 & m2;
          const uint32_t* off = a.cov.off[p12];
          uint32_t is, iv;
          if (nsc1 == 1) {
            const int istar = sc1a ? __ffs(sc1a) - 1 : 32 + __ffs(sc1b) - 1;
            is = off[0] + istar; iv = off[1] + istar;
          } else {
            is = off[2]; iv = off[3];
          }
          if (lane == 0) {
            if (sc2 && (s_cov[is] & sc2) != sc2) atomicOr(&s_cov[is], sc2);
            if (vc2 && (s_cov[iv] & vc2) != vc2) atomicOr(&s_cov[iv], vc2);
          }
        }
      }
      if (p23 >= 0 && nsc2 <= 1) {
        bool cond = nsc2 == 1;
        if (!cond) cond = __reduce_max_sync(0xffffffffu, in2 ? iabs_u(u2 - ub2) : 0u) >= th2;
        if (cond) {
          const uint32_t sc3 = (__ballot_sync(0xffffffffu, u3 >= 0) & m3) ^ sb3;
          const uint32_t vc3 = __ballot_sync(0xffffffffu, in3 && iabs_u(u3 - ub3) >= (uint32_t)tg3) & ~sc3 & m3;
          const uint32_t* off = a.cov.off[p23];
          uint32_t is, iv;
          if (nsc2 == 1) {
            const int istar = __ffs(sc2) - 1;
            is = off[0] + istar; iv = off[1] + istar;
          } else {
            is = off[2]; iv = off[3];
          }
          if (lane == 0) {
            if (sc3 && (s_cov[is] & sc3) != sc3) atomicOr(&s_cov[is], sc3);
            if (vc3 && (s_cov[iv] & vc3) != vc3) atomicOr(&s_cov[iv], vc3);
          }
        }
      }
    }
    my_chk += (unsigned long long)ncand;
  }
  // ---- a9: block then global reductions (every lane of a warp holds the same counts)
  if (lane == 0) {
    atomicAdd(&s_cnt[0], my_chk);
    atomicAdd(&s_cnt[1], my_v);
    atomicMin(&s_cex, my_cex);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&a.res.checked[b]), s_cnt[0]);
    atomicAdd(reinterpret_cast<unsigned long long*>(&a.res.violated[b]), s_cnt[1]);
    if (s_cex != kNone) {
      atomicMin(reinterpret_cast<unsigned long long*>(&a.res.first_cex[b]), s_cex);
      atomicMin(reinterpret_cast<unsigned long long*>(&a.res.first_cex_unflagged[b]), s_cex);
    }
  }
  for (uint32_t w = threadIdx.x; w < nw; w += blockDim.x)
    if (s_cov[w]) { atomicOr(&a.res.cov_all[w], s_cov[w]); atomicOr(&a.res.cov_certain[w], s_cov[w]); }
}

}  // namespace kw

// the warp-per-candidate kernel when it applies (int8, 3 layers, widths <= 64 / 32 / 32, subset
// spaces, a plain check); *supported = false otherwise (the caller takes k_small)
cudaError_t launch_warp3(const DevNet& net, int n_base, const DevPert& pert, const DevProp& prop, const DevCov& cov,
                         const DevResult& res, BaseWS ws, int num_sms, cudaStream_t st, bool* supported) {
  *supported = net.numeric == MLPV_NUM_INT8 && net.L == 3 && net.sizes[1] <= 64 && net.sizes[2] <= 32 &&
               net.sizes[3] <= 32 && (pert.kind == MLPV_PERT_SUBSET_REPLACE || pert.kind == MLPV_PERT_SUBSET_OFFSET) &&
               !pert.restrict_on && pert.n_steps == 0 && pert.n_pixels >= 2 && cov.n_words <= 256 && ws.delta != nullptr;
  if (!*supported) return cudaSuccess;
  kw::Args a;
  a.net = net; a.pert = pert; a.prop = prop; a.cov = cov; a.res = res; a.ws = ws;
  const uint64_t len = pert.end - pert.begin;
  const uint64_t nchunk = (len + kw::kChunk - 1) / kw::kChunk;
  // ~8 resident blocks per SM overall (registers: ~64 per thread)
  uint64_t gx = (uint64_t)(12 * num_sms + n_base - 1) / (uint64_t)n_base;
  const uint64_t need = (nchunk + kw::kWarps - 1) / kw::kWarps;
  if (gx > need) gx = need;
  if (gx < 1) gx = 1;
  // ~12 resident blocks per SM overall (3 per SM by the launch bounds)
  if (net.sizes[1] == 64 && net.sizes[2] == 32) kw::k_warp3<true><<<dim3((unsigned)gx, (unsigned)n_base), 32 * kw::kWarps, 0, st>>>(a);
  else kw::k_warp3<false><<<dim3((unsigned)gx, (unsigned)n_base), 32 * kw::kWarps, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace mlpv
