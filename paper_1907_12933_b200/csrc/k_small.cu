// k_small.cu -- CUDA-core kernels for subset / tuple perturbation spaces of small nets
// (BASELINE configs 1-3) and the per-base prologue (K0) shared by every path.
//
// Hot path per candidate (one thread = one candidate):
//   a2 decode the index (pair rank / mixed radix, reading C14)
//   a4 layer 1 as a rank-|S| update of the base potentials, u1 = u1_base + sum_k Delta[k][l_k]
//      (Eq. 1; exact in Z/2^32 for the fixed-point numerics)
//   a5/a6 hidden activation (Eq. 2 sigmoid, PL-sigmoid C17, ReLU+requant C18) and the remaining
//      dense layers on CUDA cores (FFMA / IMAD / DP4A) with weights resident in shared memory
//   a7 argmax (lowest index on ties), top-2 margin, property
//   a8 sign / value / distance predicates and SS / SV / VS / VV pair bits
//   a9 block-level reduction of counts, lowest-index counterexample and coverage words.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "mlpv_internal.cuh"

namespace mlpv {

// --------------------------------------------------------------------------- numeric traits
template <int NUM> struct NT;
template <> struct NT<MLPV_NUM_FP32> { using P = float; };   // potential type
template <> struct NT<MLPV_NUM_Q4_12> { using P = int32_t; };
template <> struct NT<MLPV_NUM_INT8> { using P = int32_t; };

__device__ __forceinline__ float wload_f(const void* W, int numeric, size_t i) {
  if (numeric == MLPV_NUM_FP32) return static_cast<const float*>(W)[i];
  // bf16 bits -> fp32 (exact)
  return __uint_as_float(static_cast<uint32_t>(static_cast<const uint16_t*>(W)[i]) << 16);
}
__device__ __forceinline__ int32_t wload_i(const void* W, int numeric, size_t i) {
  if (numeric == MLPV_NUM_Q4_12) return static_cast<const int16_t*>(W)[i];
  return static_cast<const int8_t*>(W)[i];
}
// lane's partial dot product of weight row `row` (fan-in `fan`) with the activations in shared
// memory: 8 bf16 / 16 int8 weights per 16-byte load when the row allows it, element-wise otherwise
__device__ __forceinline__ float row_dot_f(const void* W, int numeric, int row, int fan, const float* h, int lane) {
  float acc = 0.f;
  if (numeric == MLPV_NUM_BF16 && (fan & 7) == 0) {
    const uint4* wr = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(W) + (size_t)row * fan);
    for (int q = lane; q < (fan >> 3); q += 32) {
      const uint4 w8 = __ldg(wr + q);
      const float4 h0 = reinterpret_cast<const float4*>(h)[2 * q], h1 = reinterpret_cast<const float4*>(h)[2 * q + 1];
      acc = fmaf(__uint_as_float(w8.x << 16), h0.x, acc);
      acc = fmaf(__uint_as_float(w8.x & 0xFFFF0000u), h0.y, acc);
      acc = fmaf(__uint_as_float(w8.y << 16), h0.z, acc);
      acc = fmaf(__uint_as_float(w8.y & 0xFFFF0000u), h0.w, acc);
      acc = fmaf(__uint_as_float(w8.z << 16), h1.x, acc);
      acc = fmaf(__uint_as_float(w8.z & 0xFFFF0000u), h1.y, acc);
      acc = fmaf(__uint_as_float(w8.w << 16), h1.z, acc);
      acc = fmaf(__uint_as_float(w8.w & 0xFFFF0000u), h1.w, acc);
    }
    return acc;
  }
  for (int j = lane; j < fan; j += 32) acc = fmaf(wload_f(W, numeric, (size_t)row * fan + j), h[j], acc);
  return acc;
}
__device__ __forceinline__ int32_t row_dot_i(const void* W, int numeric, int row, int fan, const int32_t* h, int lane) {
  int32_t acc = 0;
  for (int j = lane; j < fan; j += 32) acc += wload_i(W, numeric, (size_t)row * fan + j) * h[j];
  return acc;
}
// Base-prologue dots, four weight rows per warp at once: lane-contiguous 32-bit weight words (one
// 128-byte load per row and warp), so the shared-memory reads of the input vector are conflict-free
// and each of them serves four rows (a 16-byte-per-lane row layout made the reads 16-way bank
// conflicted and the prologue shared-memory bound).  Rows >= nrows contribute nothing.
// bf16 rows (fan even) x double h (+ org): fp64 sums, two chains per row.
__device__ __forceinline__ void rows4_bf16_d(const uint16_t* W, int fan, int r0, int nrows, const double* h, double org,
                                             int lane, double (&acc)[4]) {
  const int nw2 = fan >> 1;
  const uint32_t* wr[4];
  bool ok[4];
#pragma unroll
  for (int r = 0; r < 4; r++) {
    ok[r] = r0 + r < nrows;
    wr[r] = reinterpret_cast<const uint32_t*>(W + (size_t)(ok[r] ? r0 + r : r0) * fan);
  }
  double a[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  const double2* h2 = reinterpret_cast<const double2*>(h);
#pragma unroll 4
  for (int w = lane; w < nw2; w += 32) {
    const double2 hh = h2[w];
    const double x0 = hh.x + org, x1 = hh.y + org;
#pragma unroll
    for (int r = 0; r < 4; r++)
      if (ok[r]) {
        const uint32_t q = __ldg(wr[r] + w);
        a[r][0] = fma((double)__uint_as_float(q << 16), x0, a[r][0]);
        a[r][1] = fma((double)__uint_as_float(q & 0xFFFF0000u), x1, a[r][1]);
      }
  }
#pragma unroll
  for (int r = 0; r < 4; r++) acc[r] = a[r][0] + a[r][1];
}
// int8 rows (fan % 4 == 0) x int32 h (u8 values): exact int32 sums
__device__ __forceinline__ void rows4_i8(const int8_t* W, int fan, int r0, int nrows, const int32_t* h, int lane,
                                         int32_t (&acc)[4]) {
  const int nw4 = fan >> 2;
  const uint32_t* wr[4];
  bool ok[4];
#pragma unroll
  for (int r = 0; r < 4; r++) {
    ok[r] = r0 + r < nrows;
    wr[r] = reinterpret_cast<const uint32_t*>(W + (size_t)(ok[r] ? r0 + r : r0) * fan);
    acc[r] = 0;
  }
  const int4* h4 = reinterpret_cast<const int4*>(h);
#pragma unroll 4
  for (int w = lane; w < nw4; w += 32) {
    const int4 hh = h4[w];
#pragma unroll
    for (int r = 0; r < 4; r++)
      if (ok[r]) {
        const uint32_t q = __ldg(wr[r] + w);
        acc[r] += (int32_t)(int8_t)q * hh.x + (int32_t)(int8_t)(q >> 8) * hh.y + (int32_t)(int8_t)(q >> 16) * hh.z +
                  (int32_t)(int8_t)(q >> 24) * hh.w;
      }
  }
}
__device__ __forceinline__ float in_f(const void* x, int numeric, size_t i) {
  if (numeric == MLPV_NUM_FP32) return static_cast<const float*>(x)[i];
  return __uint_as_float(static_cast<uint32_t>(static_cast<const uint16_t*>(x)[i]) << 16);
}
__device__ __forceinline__ int32_t in_i(const void* x, int numeric, size_t i) {
  if (numeric == MLPV_NUM_Q4_12) return static_cast<const int16_t*>(x)[i];
  return static_cast<const uint8_t*>(x)[i];
}
__device__ __forceinline__ float lvl_f(const void* lv, int numeric, int q) {
  if (numeric == MLPV_NUM_FP32) return static_cast<const float*>(lv)[q];
  return __uint_as_float(static_cast<uint32_t>(static_cast<const uint16_t*>(lv)[q]) << 16);
}
__device__ __forceinline__ int32_t lvl_i(const void* lv, int q) { return static_cast<const int16_t*>(lv)[q]; }

// C17 piecewise-linear sigmoid on a Q4.12 potential
__device__ __forceinline__ int32_t pl_sigmoid(const int16_t* T, int32_t u16) {
  int32_t t = u16 + 32768;
  int32_t i = t >> 9, f = t & 511;
  int32_t y0 = T[i], y1 = T[i + 1];
  return y0 + (((y1 - y0) * f + 256) >> 9);
}

// hidden activation of a fixed-point potential (C16 / C18)
__device__ __forceinline__ int32_t act_fixed(int numeric, int act, int32_t acc, int sh, const int16_t* knots) {
  if (numeric == MLPV_NUM_Q4_12) {
    int32_t u16 = (acc + 2048) >> 12;                 // arithmetic shift = floor; round half up
    u16 = max(-32768, min(32767, u16));
    return act == MLPV_ACT_PL_SIGMOID ? pl_sigmoid(knots, u16) : max(u16, 0);
  }
  int32_t r = sh > 0 ? (1 << (sh - 1)) : 0;
  return max(0, min(255, (acc + r) >> sh));
}

__device__ __forceinline__ float act_float(int act, float u) {
  return act == MLPV_ACT_SIGMOID ? 1.0f / (1.0f + expf(-u)) : fmaxf(u, 0.0f);   // Eq. 2
}

// --------------------------------------------------------------------------- K0: base prologue
// One CTA per base input: full forward of the base image (same arithmetic as the candidates for
// the fixed-point numerics, fp32 for the float numerics), base class, and the layer-1 delta
// tables Delta[s][l][i] = W1[i, p_s] * (x'_{p_s}(l) - x_{p_s}) of subset / tuple spaces.
__global__ void k_base_prologue(DevNet net, const void* bases, DevPert pert, const void* levels, BaseWS ws) {
  extern __shared__ __align__(16) double sm_d[];
  const int b = blockIdx.x;
  const int n0 = net.sizes[0];
  int maxw = 0;
  for (int l = 0; l <= net.L; l++) maxw = max(maxw, net.sizes[l]);
  // float numerics: the base trace in double (every potential rounded to fp32 once; reading C19 /
  // C23: the float kernels take the base potentials as their reference point)
  double* hf = sm_d;                              // [maxw]
  double* hn = sm_d + maxw;                       // [maxw]
  int32_t* hi = reinterpret_cast<int32_t*>(sm_d);
  int32_t* hin = reinterpret_cast<int32_t*>(sm_d + maxw);
  const bool fixed = net.numeric == MLPV_NUM_Q4_12 || net.numeric == MLPV_NUM_INT8;
  const size_t in_sz = net.numeric == MLPV_NUM_FP32 ? 4 : (net.numeric == MLPV_NUM_INT8 ? 1 : 2);
  const char* x = static_cast<const char*>(bases) + in_sz * (size_t)n0 * b;
  bool badq = false;
  for (int j = threadIdx.x; j < n0; j += blockDim.x) {
    if (fixed) {
      hi[j] = in_i(x, net.numeric, j);
      if (net.numeric == MLPV_NUM_Q4_12 && (hi[j] < 0 || hi[j] > 4096)) badq = true;   // reading C16
    } else {
      hf[j] = in_f(x, net.numeric, j);
    }
  }
  if (badq && ws.status) atomicOr(ws.status, kStatusQ412Base);
  __syncthreads();
  // dense layers: one warp per output neuron, lanes stride the fan-in (coalesced weight rows),
  // warp-shuffle sums
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const bool l1_clamp = ws.base1 != nullptr && pert.kind == MLPV_PERT_PHILOX_CLAMP && !fixed;
  if (ws.base1 != nullptr) {                        // PHILOX_BOX: W1 x + b1 + origin W1 1 (fp64 sum)
    const int n1 = net.sizes[1];                    // PHILOX_CLAMP: W1 x + b1 (origin enters via d)
    const double org = pert.kind == MLPV_PERT_PHILOX_BOX ? pert.origin_d : 0.0;
    for (int i0 = 4 * wid; i0 < n1; i0 += 4 * nw) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      if (net.numeric == MLPV_NUM_BF16 && (n0 & 1) == 0) {
        rows4_bf16_d(static_cast<const uint16_t*>(net.W[0]), n0, i0, n1, hf, org, lane, acc);
      } else {
        for (int r = 0; r < 4 && i0 + r < n1; r++)
          for (int j = lane; j < n0; j += 32)
            acc[r] += (double)wload_f(net.W[0], net.numeric, (size_t)(i0 + r) * n0 + j) * ((double)hf[j] + org);
      }
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
      if (lane < 4 && i0 + lane < n1) {
        const int i = i0 + lane;
        const double v = (lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3]) +
                         (double)static_cast<const float*>(net.b[0])[i];
        const float u = (float)v;
        ws.base1[(size_t)b * n1 + i] = u;
        if (l1_clamp) {
          // PHILOX_CLAMP: this sum is the base's layer-1 potential itself (reading C23), so the
          // dense loop below starts at layer 2
          static_cast<float*>(ws.trace)[(size_t)b * net.trace_len + net.loff[1] + i] = u;
          if (net.L > 1) hn[i] = net.act == MLPV_ACT_SIGMOID ? 1.0 / (1.0 + exp(-v)) : (v > 0.0 ? v : 0.0);
        }
      }
    }
  }
  if (ws.clampc != nullptr) {
    // PHILOX_CLAMP clamp bounds of every pixel for k_fused3's generator: d = min(max(off, -x), 1 - x)
    // in units of 2^-s, as fp16 (RN).  The contraction is exact iff each bound is exact where it
    // can bind: -x 2^s when x <= -min(off) (x = 0, or x >= 2^(-17-s) for a bf16 x), 1 - x when
    // 1 - x <= max(off).  A pixel outside [0, 1] or with an inexact binding bound is reported
    // through the status word (mlpv_sync).
    const int nch = (n0 + 7) / 8;
    const float sc = exp2f((float)pert.clamp_s);
    const double o15 = pert.origin_d + 15.0 * pert.step_d;
    const double offlo = fmin(pert.origin_d, o15), offhi = fmax(pert.origin_d, o15);
    uint32_t bad = 0;
    for (int e = threadIdx.x; e < 4 * nch; e += blockDim.x) {
      const int ch = e >> 2, k = e & 3;
      uint32_t nx2 = 0, px2 = 0;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int p = 8 * ch + 2 * k + h;
        uint16_t nx = 0, px = 0;
        if (p < n0) {
          const float xv = (float)hf[p];
          const __half hn = __float2half_rn(-xv * sc), hp = __float2half_rn((1.0f - xv) * sc);
          nx = __half_as_ushort(hn);
          px = __half_as_ushort(hp);
          if (!(xv >= 0.0f && xv <= 1.0f)) bad = 1;
          if ((double)xv <= -offlo && __half2float(hn) != -xv * sc) bad = 1;         // the lower bound binds
          if (1.0 - (double)xv <= offhi && __half2float(hp) != (1.0f - xv) * sc) bad = 1;   // the upper one
        }
        nx2 |= (uint32_t)nx << (16 * h);
        px2 |= (uint32_t)px << (16 * h);
      }
      uint32_t* dst = reinterpret_cast<uint32_t*>(ws.clampc + (size_t)b * 2 * nch + 2 * ch);
      dst[k] = nx2;
      dst[4 + k] = px2;
    }
    if (bad) atomicOr(ws.status, kStatusClampBase);
  }
  const int T = net.trace_len;
  if (l1_clamp) {                                   // layer 1 done above (hn holds its activations)
    __syncthreads();
    if (net.L > 1) {
      for (int i = threadIdx.x; i < net.sizes[1]; i += blockDim.x) hf[i] = hn[i];
      __syncthreads();
    }
  }
  for (int l = l1_clamp ? 2 : 1; l <= net.L; l++) {
    const int nl = net.sizes[l], fan = net.sizes[l - 1];
    for (int i0 = 4 * wid; i0 < nl; i0 += 4 * nw) {
      if (fixed) {
        int32_t acc[4] = {0, 0, 0, 0};
        if (net.numeric == MLPV_NUM_INT8 && (fan & 3) == 0) {
          rows4_i8(static_cast<const int8_t*>(net.W[l - 1]), fan, i0, nl, hi, lane, acc);
        } else {
          for (int r = 0; r < 4 && i0 + r < nl; r++) acc[r] = row_dot_i(net.W[l - 1], net.numeric, i0 + r, fan, hi, lane);
        }
#pragma unroll
        for (int r = 0; r < 4; r++) acc[r] = __reduce_add_sync(0xffffffffu, acc[r]);
        if (lane < 4 && i0 + lane < nl) {
          const int i = i0 + lane;
          const int32_t v = (lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3]) +
                            static_cast<const int32_t*>(net.b[l - 1])[i];
          static_cast<int32_t*>(ws.trace)[(size_t)b * T + net.loff[l] + i] = v;
          if (l < net.L) hin[i] = act_fixed(net.numeric, net.act, v, net.shift[l - 1], net.knots);
        }
      } else {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        if (net.numeric == MLPV_NUM_BF16 && (fan & 1) == 0) {
          rows4_bf16_d(static_cast<const uint16_t*>(net.W[l - 1]), fan, i0, nl, hf, 0.0, lane, acc);
        } else {
          for (int r = 0; r < 4 && i0 + r < nl; r++)
            for (int j = lane; j < fan; j += 32)
              acc[r] += (double)wload_f(net.W[l - 1], net.numeric, (size_t)(i0 + r) * fan + j) * hf[j];
        }
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
        if (lane < 4 && i0 + lane < nl) {
          const int i = i0 + lane;
          const double v = (lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3]) +
                           (double)static_cast<const float*>(net.b[l - 1])[i];
          static_cast<float*>(ws.trace)[(size_t)b * T + net.loff[l] + i] = (float)v;
          if (l < net.L) hn[i] = net.act == MLPV_ACT_SIGMOID ? 1.0 / (1.0 + exp(-v)) : (v > 0.0 ? v : 0.0);
        }
      }
    }
    __syncthreads();
    if (l < net.L) {
      for (int i = threadIdx.x; i < nl; i += blockDim.x) {
        if (fixed) hi[i] = hin[i]; else hf[i] = hn[i];
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    const int nL = net.sizes[net.L];
    int c = 0;
    if (fixed) {
      const int32_t* y = static_cast<const int32_t*>(ws.trace) + (size_t)b * T + net.loff[net.L];
      for (int i = 1; i < nL; i++) if (y[i] > y[c]) c = i;
    } else {
      const float* y = static_cast<const float*>(ws.trace) + (size_t)b * T + net.loff[net.L];
      for (int i = 1; i < nL; i++) if (y[i] > y[c]) c = i;
    }
    ws.cls[b] = c;
  }
  // delta tables (subset / tuple spaces only)
  if (ws.delta == nullptr) return;
  const int n1 = net.sizes[1], q = pert.n_levels, S = ws.S;
  const size_t per_base = (size_t)S * q * n1;
  for (size_t e = threadIdx.x; e < per_base; e += blockDim.x) {
    const int i = (int)(e % n1);
    const int lq = (int)((e / n1) % q);
    const int s = (int)(e / ((size_t)n1 * q));
    const int p = pert.kind == MLPV_PERT_TUPLE_REPLACE ? s : pert.pixels[s];
    if (fixed) {
      const int32_t xp = in_i(x, net.numeric, p);
      int32_t xn;
      if (pert.kind == MLPV_PERT_SUBSET_OFFSET) {
        const int32_t hi_ = net.numeric == MLPV_NUM_Q4_12 ? 4096 : 255;
        xn = max(0, min(hi_, xp + lvl_i(levels, lq)));
      } else {
        xn = lvl_i(levels, lq);
      }
      static_cast<int32_t*>(ws.delta)[(size_t)b * per_base + e] = wload_i(net.W[0], net.numeric, (size_t)i * n0 + p) * (xn - xp);
    } else {
      const float xp = in_f(x, net.numeric, p);
      const float xn = lvl_f(levels, net.numeric, lq);
      static_cast<float*>(ws.delta)[(size_t)b * per_base + e] = wload_f(net.W[0], net.numeric, (size_t)i * n0 + p) * (xn - xp);
    }
  }
}

cudaError_t launch_base_prologue(const DevNet& net, const void* bases, int n_base, const DevPert& pert,
                                 const void* levels_dev, BaseWS ws, cudaStream_t st) {
  int maxw = 0;
  for (int l = 0; l <= net.L; l++) maxw = maxw > net.sizes[l] ? maxw : net.sizes[l];
  size_t smem = sizeof(double) * 2 * (size_t)maxw;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_base_prologue, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_base_prologue<<<n_base, 256, smem, st>>>(net, bases, pert, levels_dev, ws);
  return cudaGetLastError();
}

// --------------------------------------------------------------------------- K1: small-net kernel
struct SmallArgs {
  DevNet net;
  DevPert pert;
  DevProp prop;
  DevCov cov;
  DevResult res;
  BaseWS ws;
  int n_base;
  const uint64_t* eval_idx;   // eval mode: candidate indices of base eval_base
  int64_t eval_n;
  int eval_base;
  void* eval_out;             // [eval_n x T]
  int tbl_in_smem;            // delta table of the block's base staged in smem
  int ds;                     // row stride of the delta table as read: n1 (global) or n1 | 1 (smem:
                              // an odd stride puts the rows the lanes of a warp read in different banks)
  const void* bases;          // [n_base x n_0] base images (restriction R)
};

// Restriction R of checkNN (reading C27): delta(I^d, I) <= b over the changed
// pixels (the others contribute 0): fixed point exactly in int64 against floor(b^2 S^2), float
// in double in ascending pixel order (the order of the oracle's plain sum), no contraction.
__device__ __forceinline__ double sq_rn(double d) { return __dmul_rn(d, d); }

__device__ __forceinline__ uint32_t dp4a_us(uint32_t a_u8x4, uint32_t b_s8x4, int32_t c) {
  int32_t d;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a_u8x4), "r"(b_s8x4), "r"(c));
  return (uint32_t)d;
}

// pair rank -> (i, j), i < j < n0, lexicographic (i outer)
__device__ __forceinline__ void unrank_pair(uint32_t pr, int n0, int& i, int& j) {
  // cum(i) = i*(2*n0 - i - 1)/2 pairs precede row i
  const double a = 2.0 * n0 - 1.0;
  int ii = (int)floor((a - sqrt(a * a - 8.0 * (double)pr)) * 0.5);
  ii = max(0, min(n0 - 2, ii));
  auto cum = [n0](int r) -> uint32_t { return (uint32_t)((int64_t)r * (2 * n0 - r - 1) / 2); };
  while (ii + 1 <= n0 - 2 && cum(ii + 1) <= pr) ii++;
  while (ii > 0 && cum(ii) > pr) ii--;
  i = ii;
  j = ii + 1 + (int)(pr - cum(ii));
}

template <typename P>
__device__ __forceinline__ bool sgn(P u) { return u >= P(0); }

// Coverage of one pair (k, k+1) for one candidate; bits OR-ed into the block's smem words.
// lo/up: candidate potentials; blo/bup: base potentials (smem).  Float numerics also evaluate
// the ambiguity of the predicates used (reading C20) to decide cov_certain.
template <typename P, int ML, int MU>
__device__ __forceinline__ void cover_pair(const P (&lo)[ML], const P (&up)[MU], const P* blo, const P* bup,
                                           int nlo, int nup, P tg, P th, float tau_lo, float tau_up,
                                           uint32_t* sm_all, uint32_t* sm_cert, const uint32_t off[4], bool fl) {
  int nsc = 0, istar = -1;
  P linf = P(0);
#pragma unroll
  for (int i = 0; i < ML; i++) {
    if (i < nlo) {
      const bool c = sgn(lo[i]) != sgn(blo[i]);
      if (c) { if (istar < 0) istar = i; nsc++; }
      P d = lo[i] - blo[i];
      d = d < P(0) ? -d : d;
      linf = d > linf ? d : linf;
    }
  }
  const bool dc = (nsc == 0) && (linf >= th);
  if (!(nsc == 1 || dc)) return;           // no cover of this pair can hold
  // ambiguity (float numerics)
  bool amb = false;
  if (fl) {
#pragma unroll
    for (int i = 0; i < ML; i++)
      if (i < nlo && (fabsf((float)lo[i]) < tau_lo || fabsf((float)blo[i]) < tau_lo)) amb = true;
    if (nsc == 0 && fabsf((float)(linf - th)) < tau_lo) amb = true;
  }
  const int wpr = (nup + 31) >> 5;
#pragma unroll
  for (int j = 0; j < MU; j++) {
    if (j < nup) {
      const bool sc = sgn(up[j]) != sgn(bup[j]);
      P d = up[j] - bup[j];
      d = d < P(0) ? -d : d;
      const bool vc = !sc && d >= tg;
      if (fl && (fabsf((float)up[j]) < tau_up || fabsf((float)bup[j]) < tau_up || fabsf((float)(d - tg)) < tau_up)) amb = true;
      const uint32_t bit = 1u << (j & 31);
      const int wj = j >> 5;
      if (nsc == 1) {
        if (sc) atomicOr(&sm_all[off[0] + istar * wpr + wj], bit);
        if (vc) atomicOr(&sm_all[off[1] + istar * wpr + wj], bit);
      } else {
        if (sc) atomicOr(&sm_all[off[2] + wj], bit);
        if (vc) atomicOr(&sm_all[off[3] + wj], bit);
      }
    }
  }
  if (fl && !amb) {
    // replay the same bits into the certain set
#pragma unroll
    for (int j = 0; j < MU; j++) {
      if (j < nup) {
        const bool sc = sgn(up[j]) != sgn(bup[j]);
        P d = up[j] - bup[j];
        d = d < P(0) ? -d : d;
        const bool vc = !sc && d >= tg;
        const uint32_t bit = 1u << (j & 31);
        const int wj = j >> 5;
        if (nsc == 1) {
          if (sc) atomicOr(&sm_cert[off[0] + istar * wpr + wj], bit);
          if (vc) atomicOr(&sm_cert[off[1] + istar * wpr + wj], bit);
        } else {
          if (sc) atomicOr(&sm_cert[off[2] + wj], bit);
          if (vc) atomicOr(&sm_cert[off[3] + wj], bit);
        }
      }
    }
  }
}

// Dense layer l >= 2 on CUDA cores: u[i] = b[i] + sum_j W[i][j] h[j]
template <int NUM, int MI, int MO>
__device__ __forceinline__ void dense(typename NT<NUM>::P (&u)[MO], const float (&hf)[MI], const int32_t (&hi)[MI],
                                      const uint32_t (&hp)[(MI + 3) / 4], const void* Wsm, const void* bsm,
                                      int nin, int nout) {
  if constexpr (NUM == MLPV_NUM_FP32) {
    const float* W = static_cast<const float*>(Wsm);
#pragma unroll
    for (int i = 0; i < MO; i++) {
      if (i < nout) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < MI; j++) if (j < nin) acc = fmaf(W[i * nin + j], hf[j], acc);
        u[i] = acc + static_cast<const float*>(bsm)[i];
      }
    }
  } else if constexpr (NUM == MLPV_NUM_Q4_12) {
    const int16_t* W = static_cast<const int16_t*>(Wsm);
#pragma unroll
    for (int i = 0; i < MO; i++) {
      if (i < nout) {
        int32_t acc = static_cast<const int32_t*>(bsm)[i];
#pragma unroll
        for (int j = 0; j < MI; j++) if (j < nin) acc += (int32_t)W[i * nin + j] * hi[j];
        u[i] = acc;
      }
    }
  } else {
    // int8 rows packed as s8x4 words, row stride (nin+3)/4 words
    const uint32_t* W = static_cast<const uint32_t*>(Wsm);
    const int wpr = (nin + 3) >> 2;
#pragma unroll
    for (int i = 0; i < MO; i++) {
      if (i < nout) {
        int32_t acc = static_cast<const int32_t*>(bsm)[i];
#pragma unroll
        for (int w = 0; w < (MI + 3) / 4; w++) if (w < wpr) acc = (int32_t)dp4a_us(hp[w], W[i * wpr + w], acc);
        u[i] = acc;
      }
    }
  }
}

template <int NUM, int MI>
__device__ __forceinline__ void activate(const typename NT<NUM>::P (&u)[MI], float (&hf)[MI], int32_t (&hi)[MI],
                                         uint32_t (&hp)[(MI + 3) / 4], int n, int act, int sh, const int16_t* knots) {
  if constexpr (NUM == MLPV_NUM_FP32) {
#pragma unroll
    for (int i = 0; i < MI; i++) hf[i] = i < n ? act_float(act, u[i]) : 0.f;
  } else {
#pragma unroll
    for (int i = 0; i < MI; i++) hi[i] = i < n ? act_fixed(NUM, act, u[i], sh, knots) : 0;
    if constexpr (NUM == MLPV_NUM_INT8) {
#pragma unroll
      for (int w = 0; w < (MI + 3) / 4; w++) {
        uint32_t v = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) if (4 * w + k < MI) v |= (uint32_t)hi[4 * w + k] << (8 * k);
        hp[w] = v;
      }
    }
  }
}

// M1..M3: compile-time maxima of n_1..n_3 (register arrays); L in {2, 3}.
template <int NUM, int L, int M1, int M2, int M3>
__global__ void __launch_bounds__(256) k_small(SmallArgs a) {
  using P = typename NT<NUM>::P;
  constexpr bool FL = NUM == MLPV_NUM_FP32;
  extern __shared__ __align__(16) uint8_t smem[];
  const DevNet& net = a.net;
  const int T = net.trace_len;
  const int n0 = net.sizes[0], n1 = net.sizes[1], n2 = net.sizes[2], n3 = L == 3 ? net.sizes[3] : 0;
  const int nL = net.sizes[L];
  const bool eval = a.eval_idx != nullptr;
  const int b = eval ? a.eval_base : blockIdx.y;
  const int q = a.pert.n_levels;

  // ---- shared-memory carve-up
  uint8_t* sp = smem;
  auto take = [&](size_t bytes) { uint8_t* r = sp; sp += (bytes + 15) & ~size_t(15); return r; };
  P* s_base = reinterpret_cast<P*>(take(sizeof(P) * T));
  void* s_W2 = take(NUM == MLPV_NUM_FP32 ? 4 * (size_t)n2 * n1 : (NUM == MLPV_NUM_Q4_12 ? 2 * (size_t)n2 * n1 : 4 * (size_t)n2 * ((n1 + 3) / 4)));
  void* s_b2 = take(4 * (size_t)n2);
  void* s_W3 = take(L == 3 ? (NUM == MLPV_NUM_FP32 ? 4 * (size_t)n3 * n2 : (NUM == MLPV_NUM_Q4_12 ? 2 * (size_t)n3 * n2 : 4 * (size_t)n3 * ((n2 + 3) / 4))) : 0);
  void* s_b3 = take(L == 3 ? 4 * (size_t)n3 : 0);
  int16_t* s_knots = reinterpret_cast<int16_t*>(take(net.knots ? 129 * 2 : 0));
  uint32_t* s_cov = reinterpret_cast<uint32_t*>(take(eval ? 0 : 4 * (size_t)a.cov.n_words * (FL ? 2 : 1)));
  const size_t per_base = (size_t)a.ws.S * q * n1;
  P* s_delta = reinterpret_cast<P*>(take(a.tbl_in_smem ? sizeof(P) * (per_base / n1) * a.ds : 0));
  __shared__ unsigned long long s_cnt[3];
  __shared__ unsigned long long s_cex[2];

  // early-exit pass (NEXT-2): a base input decided at an earlier step has nothing left to check
  if (a.pert.shell > 0 && !eval) {
    const unsigned long long k = a.pert.decided[b];
    if (k != kNone && (int)(k >> kStepShift) < a.pert.shell) return;      // uniform over the block
  }
  // ---- stage per-base data
  for (int t = threadIdx.x; t < T; t += blockDim.x) s_base[t] = static_cast<const P*>(a.ws.trace)[(size_t)b * T + t];
  {
    if constexpr (NUM == MLPV_NUM_FP32) {
      for (int t = threadIdx.x; t < n2 * n1; t += blockDim.x) static_cast<float*>(s_W2)[t] = static_cast<const float*>(net.W[1])[t];
      if (L == 3) for (int t = threadIdx.x; t < n3 * n2; t += blockDim.x) static_cast<float*>(s_W3)[t] = static_cast<const float*>(net.W[2])[t];
    } else if constexpr (NUM == MLPV_NUM_Q4_12) {
      for (int t = threadIdx.x; t < n2 * n1; t += blockDim.x) static_cast<int16_t*>(s_W2)[t] = static_cast<const int16_t*>(net.W[1])[t];
      if (L == 3) for (int t = threadIdx.x; t < n3 * n2; t += blockDim.x) static_cast<int16_t*>(s_W3)[t] = static_cast<const int16_t*>(net.W[2])[t];
    } else {
      const int w1 = (n1 + 3) / 4, w2 = (n2 + 3) / 4;
      for (int t = threadIdx.x; t < n2 * w1; t += blockDim.x) {
        const int i = t / w1, w = t % w1;
        uint32_t v = 0;
        for (int k = 0; k < 4; k++) if (4 * w + k < n1) v |= (uint32_t)(uint8_t)static_cast<const int8_t*>(net.W[1])[i * n1 + 4 * w + k] << (8 * k);
        static_cast<uint32_t*>(s_W2)[t] = v;
      }
      if (L == 3)
        for (int t = threadIdx.x; t < n3 * w2; t += blockDim.x) {
          const int i = t / w2, w = t % w2;
          uint32_t v = 0;
          for (int k = 0; k < 4; k++) if (4 * w + k < n2) v |= (uint32_t)(uint8_t)static_cast<const int8_t*>(net.W[2])[i * n2 + 4 * w + k] << (8 * k);
          static_cast<uint32_t*>(s_W3)[t] = v;
        }
    }
    for (int t = threadIdx.x; t < n2; t += blockDim.x) static_cast<uint32_t*>(s_b2)[t] = static_cast<const uint32_t*>(net.b[1])[t];
    if (L == 3) for (int t = threadIdx.x; t < n3; t += blockDim.x) static_cast<uint32_t*>(s_b3)[t] = static_cast<const uint32_t*>(net.b[2])[t];
    if (net.knots) for (int t = threadIdx.x; t < 129; t += blockDim.x) s_knots[t] = net.knots[t];
    if (!eval) for (int t = threadIdx.x; t < (int)a.cov.n_words * (FL ? 2 : 1); t += blockDim.x) s_cov[t] = 0;
    if (a.tbl_in_smem)
      for (size_t t = threadIdx.x; t < per_base; t += blockDim.x)
        s_delta[(t / n1) * a.ds + t % n1] = static_cast<const P*>(a.ws.delta)[(size_t)b * per_base + t];
    if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
    if (threadIdx.x < 2) s_cex[threadIdx.x] = kNone;
  }
  __syncthreads();
  const P* delta = a.tbl_in_smem ? s_delta : static_cast<const P*>(a.ws.delta) + (size_t)b * per_base;
  const int base_cls = a.ws.cls[b];
  P tg[3], th[3];
  float tau[3];
#pragma unroll
  for (int l = 0; l < 3; l++) {
    if constexpr (FL) { tg[l] = a.cov.tg_f[l]; th[l] = a.cov.th_f[l]; }
    else { tg[l] = (P)a.cov.tg_i[l]; th[l] = (P)a.cov.th_i[l]; }
    tau[l] = a.cov.tau_dev ? a.cov.tau_dev[l] : a.cov.tau[l];
  }
  bool pair_on[2] = {false, false};
  uint32_t poff[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
  for (int p = 0; p < a.cov.n_pairs; p++) {
    const int k = a.cov.lower[p];
    if (k >= 1 && k <= 2) {
      pair_on[k - 1] = true;
      for (int m = 0; m < 4; m++) poff[k - 1][m] = a.cov.off[p][m];
    }
  }
  const uint64_t begin = a.pert.begin, end = a.pert.end;
  const uint64_t nwork = eval ? (uint64_t)a.eval_n : end - begin;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long my_chk = 0, my_v = 0, my_f = 0, my_cex = kNone, my_cexu = kNone;

  // one candidate from its layer-1 potentials U1 on (t: position in the range / the eval list)
  auto cand = [&](const uint64_t t, const uint64_t c, P (&U1)[M1]) {
    P U2[M2], U3[M3 > 0 ? M3 : 1];
    double rs2_f = 0.0;                                // squared distance to the base (restriction /
    long long rs2_i = 0;                               // incremental steps), float / fixed point
    if (a.pert.restrict_on && !eval) {
      const char* xb = static_cast<const char*>(a.bases);
      const size_t bo = (size_t)b * n0;
      bool inside;
      if (a.pert.kind == MLPV_PERT_TUPLE_REPLACE) {
        int pi = 0, pj = 0, li = 0, lj = 0;
        if (a.pert.tuple == 2) {
          const uint32_t rem = (uint32_t)(c % a.pert.q2);
          li = rem / q; lj = rem % q;
          unrank_pair((uint32_t)(c / a.pert.q2), n0, pi, pj);
        } else {
          pi = (int)(c / q); li = (int)(c % q);
        }
        if constexpr (FL) {
          double s2 = sq_rn((double)lvl_f(a.pert.levels, NUM, li) - (double)in_f(xb, NUM, bo + pi));
          if (a.pert.tuple == 2) s2 = __dadd_rn(s2, sq_rn((double)lvl_f(a.pert.levels, NUM, lj) - (double)in_f(xb, NUM, bo + pj)));
          rs2_f = s2;
          inside = s2 <= a.pert.r2_f;
        } else {
          const long long d0 = (long long)lvl_i(a.pert.levels, li) - in_i(xb, NUM, bo + pi);
          long long s2 = d0 * d0;
          if (a.pert.tuple == 2) {
            const long long d1 = (long long)lvl_i(a.pert.levels, lj) - in_i(xb, NUM, bo + pj);
            s2 += d1 * d1;
          }
          rs2_i = s2;
          inside = s2 <= a.pert.r2_raw;
        }
      } else {
        int dig[16];
        uint64_t cc = c;
        for (int k = a.pert.n_pixels - 1; k >= 0; k--) { dig[k] = (int)(cc % (uint64_t)q); cc /= (uint64_t)q; }
        if constexpr (FL) {
          double s2 = 0.0;
          for (int k = 0; k < a.pert.n_pixels; k++) {
            const int p = a.pert.pixels[k];
            s2 = __dadd_rn(s2, sq_rn((double)lvl_f(a.pert.levels, NUM, dig[k]) - (double)in_f(xb, NUM, bo + p)));
          }
          rs2_f = s2;
          inside = s2 <= a.pert.r2_f;
        } else {
          long long s2 = 0;
          const int hi = NUM == MLPV_NUM_Q4_12 ? 4096 : 255;
          for (int k = 0; k < a.pert.n_pixels; k++) {
            const int p = a.pert.pixels[k];
            const int32_t xp = in_i(xb, NUM, bo + p);
            const int32_t xn = a.pert.kind == MLPV_PERT_SUBSET_OFFSET ? max(0, min(hi, xp + lvl_i(a.pert.levels, dig[k])))
                                                                      : lvl_i(a.pert.levels, dig[k]);
            const long long d = (long long)xn - xp;
            s2 += d * d;
          }
          rs2_i = s2;
          inside = s2 <= a.pert.r2_raw;
        }
      }
      if (!inside) return;                           // outside R: no verdict, no coverage
    }
    // incremental bounds (NEXT-2): the step of the smallest ball b_i holding the candidate
    int cstep = 0;
    if (a.pert.n_steps > 0 && !eval) {
      cstep = 1;
      if constexpr (FL) { while (cstep < a.pert.n_steps && rs2_f > a.pert.step_r2_f[cstep - 1]) cstep++; }
      else { while (cstep < a.pert.n_steps && rs2_i > a.pert.step_r2_raw[cstep - 1]) cstep++; }
      if (a.pert.shell > 0 && cstep != a.pert.shell) return;   // early-exit pass: this shell only
    }
    // ---- a5/a6: hidden activations and dense layers
    {
      float h1f[M1]; int32_t h1i[M1]; uint32_t h1p[(M1 + 3) / 4];
      activate<NUM, M1>(U1, h1f, h1i, h1p, n1, net.act, net.shift[0], s_knots);
      dense<NUM, M1, M2>(U2, h1f, h1i, h1p, s_W2, s_b2, n1, n2);
    }
    if constexpr (L == 3) {
      float h2f[M2]; int32_t h2i[M2]; uint32_t h2p[(M2 + 3) / 4];
      activate<NUM, M2>(U2, h2f, h2i, h2p, n2, net.act, net.shift[1], s_knots);
      dense<NUM, M2, M3>(U3, h2f, h2i, h2p, s_W3, s_b3, n2, n3);
    }
    if (eval) {
      P* o = static_cast<P*>(a.eval_out) + t * T;
#pragma unroll
      for (int i = 0; i < M1; i++) if (i < n1) o[net.loff[1] + i] = U1[i];
#pragma unroll
      for (int i = 0; i < M2; i++) if (i < n2) o[net.loff[2] + i] = U2[i];
      if constexpr (L == 3) {
#pragma unroll
        for (int i = 0; i < M3; i++) if (i < n3) o[net.loff[3] + i] = U3[i];
      }
      return;
    }
    // ---- a7: argmax, margin, property
    const P* Y = (L == 3) ? U3 : U2;
    constexpr int MY = (L == 3) ? (M3 > 0 ? M3 : 1) : M2;
    int cls = 0;
    P top1 = Y[0];
#pragma unroll
    for (int i = 1; i < MY; i++) if (i < nL && Y[i] > top1) { top1 = Y[i]; cls = i; }
    bool viol, flag = false;
    if (a.prop.kind == MLPV_PROP_THRESHOLD_LITERAL || a.prop.kind == MLPV_PROP_THRESHOLD_LITERAL_ALL) {
      const int D = a.prop.target >= 0 ? a.prop.target : base_cls;
      const P V = FL ? (P)a.prop.V_f : (P)a.prop.V_i;
      bool any = false, all = true;
      P yD = Y[0];
#pragma unroll
      for (int i = 0; i < MY; i++) {
        if (i < nL) {
          if (i == D) yD = Y[i];
          if (i != D && Y[i] > V) any = true;
          if (i != D && !(Y[i] > V)) all = false;
          if (FL && fabsf((float)(Y[i] - V)) < a.cov.near_tie) flag = true;
        }
      }
      viol = (yD < V) && (a.prop.kind == MLPV_PROP_THRESHOLD_LITERAL_ALL ? all : any);
    } else {
      if constexpr (FL) {
        float top2 = -3.0e38f;
#pragma unroll
        for (int i = 0; i < MY; i++) if (i < nL && i != cls && Y[i] > top2) top2 = Y[i];
        if (nL > 1 && (float)top1 - top2 < a.cov.near_tie) flag = true;
      }
      viol = a.prop.kind == MLPV_PROP_TARGET_NEVER ? (cls == a.prop.target) : (cls != base_cls);
    }
    my_chk++;
    if (flag) my_f++;
    if (viol) {
      my_v++;
      unsigned long long key = c;
      if (a.pert.n_steps > 0) key |= (unsigned long long)cstep << kStepShift;   // key = (step, index)
      if (key < my_cex) my_cex = key;
      if (!flag && key < my_cexu) my_cexu = key;
    }
    // ---- a8: coverage
    uint32_t* s_cert = FL ? s_cov + a.cov.n_words : s_cov;
    if (pair_on[0])
      cover_pair<P, M1, M2>(U1, U2, s_base + net.loff[1], s_base + net.loff[2], n1, n2, tg[1], th[0], tau[0], tau[1],
                            s_cov, s_cert, poff[0], FL);
    if constexpr (L == 3) {
      if (pair_on[1])
        cover_pair<P, M2, (M3 > 0 ? M3 : 1)>(U2, U3, s_base + net.loff[2], s_base + net.loff[3], n2, n3, tg[2], th[1],
                                             tau[1], tau[2], s_cov, s_cert, poff[1], FL);
    }
  };
  // subset spaces: a thread takes whole runs of q consecutive indices, which share every digit but
  // the last -- the prefix (base + the delta rows of those digits) is summed once per run, each
  // candidate then adds one row (the order of the candidates does not change any result; fixed
  // point only, where the regrouped integer sums are exact -- the fp32 path keeps its summation order)
  const bool runs = !FL && !eval && (a.pert.kind == MLPV_PERT_SUBSET_OFFSET || a.pert.kind == MLPV_PERT_SUBSET_REPLACE) &&
                    a.pert.n_pixels >= 2 && nwork > 0;
  if (runs) {
    const uint64_t h0 = begin / (uint64_t)q, nruns = (end - 1) / (uint64_t)q - h0 + 1;
    const P* last = delta + (size_t)(a.pert.n_pixels - 1) * q * a.ds;
    for (uint64_t ru = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; ru < nruns; ru += stride) {
      const uint64_t hi = h0 + ru;
      P U1p[M1];
#pragma unroll
      for (int i = 0; i < M1; i++) U1p[i] = i < n1 ? s_base[i] : P(0);
      uint64_t cc = hi;
      for (int k = a.pert.n_pixels - 2; k >= 0; k--) {
        const int d = (int)(cc % (uint64_t)q);
        cc /= (uint64_t)q;
        const P* dk = delta + ((size_t)k * q + d) * a.ds;
#pragma unroll
        for (int i = 0; i < M1; i++) if (i < n1) U1p[i] += dk[i];
      }
      const uint64_t c0 = hi * (uint64_t)q;
      const int dlo = c0 < begin ? (int)(begin - c0) : 0;
      const int dhi = c0 + (uint64_t)q > end ? (int)(end - c0) : q;
      for (int dl = dlo; dl < dhi; dl++) {
        const P* dk = last + (size_t)dl * a.ds;
        P U1[M1];
#pragma unroll
        for (int i = 0; i < M1; i++) U1[i] = i < n1 ? U1p[i] + dk[i] : P(0);
        cand(c0 + dl - begin, c0 + dl, U1);
      }
    }
  } else
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nwork; t += stride) {
    const uint64_t c = eval ? a.eval_idx[t] : begin + t;
    // ---- a2 + a4: decode and incremental layer 1
    P U1[M1];
#pragma unroll
    for (int i = 0; i < M1; i++) U1[i] = i < n1 ? s_base[i] : P(0);
    if (a.pert.kind == MLPV_PERT_TUPLE_REPLACE) {
      if (a.pert.tuple == 2) {
        const uint32_t pr = (uint32_t)(c / a.pert.q2);
        const uint32_t rem = (uint32_t)(c % a.pert.q2);
        const int li = rem / q, lj = rem % q;
        int pi, pj;
        unrank_pair(pr, n0, pi, pj);
        const P* d0 = delta + ((size_t)pi * q + li) * a.ds;
        const P* d1 = delta + ((size_t)pj * q + lj) * a.ds;
#pragma unroll
        for (int i = 0; i < M1; i++) if (i < n1) U1[i] = U1[i] + d0[i] + d1[i];
      } else {
        const int pi = (int)(c / q), li = (int)(c % q);
        const P* d0 = delta + ((size_t)pi * q + li) * a.ds;
#pragma unroll
        for (int i = 0; i < M1; i++) if (i < n1) U1[i] = U1[i] + d0[i];
      }
    } else {
      // mixed-radix digits, least significant first: shifts for a power-of-two q, 32-bit
      // division when the index fits, 64-bit otherwise (warp-uniform choice)
      const int qb = __ffs(q) - 1;
      if ((q & (q - 1)) == 0) {
        uint64_t cc = c;
        for (int k = a.pert.n_pixels - 1; k >= 0; k--) {
          const int d = (int)(cc & (uint64_t)(q - 1));
          cc >>= qb;
          const P* dk = delta + ((size_t)k * q + d) * a.ds;
#pragma unroll
          for (int i = 0; i < M1; i++) if (i < n1) U1[i] += dk[i];
        }
      } else if (c < (1ull << 32)) {
        uint32_t cc = (uint32_t)c;
        for (int k = a.pert.n_pixels - 1; k >= 0; k--) {
          const int d = (int)(cc % (uint32_t)q);
          cc /= (uint32_t)q;
          const P* dk = delta + ((size_t)k * q + d) * a.ds;
#pragma unroll
          for (int i = 0; i < M1; i++) if (i < n1) U1[i] += dk[i];
        }
      } else {
        uint64_t cc = c;
        for (int k = a.pert.n_pixels - 1; k >= 0; k--) {
          const int d = (int)(cc % (uint64_t)q);
          cc /= (uint64_t)q;
          const P* dk = delta + ((size_t)k * q + d) * a.ds;
#pragma unroll
          for (int i = 0; i < M1; i++) if (i < n1) U1[i] += dk[i];
        }
      }
    }
    cand(t, c, U1);
  }
  if (eval) return;
  // ---- a9: block reduction
  const unsigned full = 0xffffffffu;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    my_chk += __shfl_xor_sync(full, my_chk, o);
    my_v += __shfl_xor_sync(full, my_v, o);
    my_f += __shfl_xor_sync(full, my_f, o);
    unsigned long long x = __shfl_xor_sync(full, my_cex, o);
    my_cex = x < my_cex ? x : my_cex;
    x = __shfl_xor_sync(full, my_cexu, o);
    my_cexu = x < my_cexu ? x : my_cexu;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s_cnt[0], my_chk);
    atomicAdd(&s_cnt[1], my_v);
    atomicAdd(&s_cnt[2], my_f);
    atomicMin(&s_cex[0], my_cex);
    atomicMin(&s_cex[1], my_cexu);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&a.res.checked[b]), s_cnt[0]);
    atomicAdd(reinterpret_cast<unsigned long long*>(&a.res.violated[b]), s_cnt[1]);
    atomicAdd(reinterpret_cast<unsigned long long*>(&a.res.flagged[b]), s_cnt[2]);
    if (s_cex[0] != kNone) atomicMin(reinterpret_cast<unsigned long long*>(&a.res.first_cex[b]), s_cex[0]);
    if (s_cex[1] != kNone) atomicMin(reinterpret_cast<unsigned long long*>(&a.res.first_cex_unflagged[b]), s_cex[1]);
  }
  for (int w = threadIdx.x; w < (int)a.cov.n_words; w += blockDim.x) {
    if (s_cov[w]) atomicOr(&a.res.cov_all[w], s_cov[w]);
    if (FL) { if (s_cov[a.cov.n_words + w]) atomicOr(&a.res.cov_certain[w], s_cov[a.cov.n_words + w]); }
    else if (s_cov[w]) atomicOr(&a.res.cov_certain[w], s_cov[w]);
  }
}

template <int NUM, int L, int M1, int M2, int M3>
static cudaError_t run_small(SmallArgs& a, int num_sms, cudaStream_t st) {
  using P = typename NT<NUM>::P;
  const DevNet& net = a.net;
  const int n1 = net.sizes[1], n2 = net.sizes[2], n3 = L == 3 ? net.sizes[3] : 0;
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  size_t smem = al(sizeof(P) * net.trace_len);
  smem += al(NUM == MLPV_NUM_FP32 ? 4 * (size_t)n2 * n1 : (NUM == MLPV_NUM_Q4_12 ? 2 * (size_t)n2 * n1 : 4 * (size_t)n2 * ((n1 + 3) / 4)));
  smem += al(4 * (size_t)n2);
  if (L == 3) {
    smem += al(NUM == MLPV_NUM_FP32 ? 4 * (size_t)n3 * n2 : (NUM == MLPV_NUM_Q4_12 ? 2 * (size_t)n3 * n2 : 4 * (size_t)n3 * ((n2 + 3) / 4)));
    smem += al(4 * (size_t)n3);
  }
  if (net.knots) smem += al(129 * 2);
  const bool eval = a.eval_idx != nullptr;
  if (!eval) smem += al(4 * (size_t)a.cov.n_words * (NUM == MLPV_NUM_FP32 ? 2 : 1));
  const int n1s = n1 | 1;
  const size_t tbl = sizeof(P) * (size_t)a.ws.S * a.pert.n_levels * n1s;
  a.tbl_in_smem = (smem + al(tbl) <= 160 * 1024) ? 1 : 0;
  a.ds = a.tbl_in_smem ? n1s : n1;
  if (a.tbl_in_smem) smem += al(tbl);
  if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
  auto kern = k_small<NUM, L, M1, M2, M3>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int threads = 256;
  dim3 grid;
  if (eval) {
    grid = dim3((unsigned)((a.eval_n + threads - 1) / threads), 1);
  } else {
    const uint64_t range = a.pert.end - a.pert.begin;
    const uint64_t need = (range + threads * 8 - 1) / (threads * 8);     // >= 8 candidates per thread
    const int want = (4 * num_sms + a.n_base - 1) / a.n_base;             // ~4 waves of CTAs overall
    uint64_t gx = need < (uint64_t)want ? need : (uint64_t)want;
    if (gx < 1) gx = 1;
    grid = dim3((unsigned)gx, (unsigned)a.n_base);
  }
  if (grid.x == 0) return cudaSuccess;
  kern<<<grid, threads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_small(const DevNet& net, const void* bases, int n_base, const DevPert& pert,
                         const DevProp& prop, const DevCov& cov, const DevResult& res, BaseWS ws,
                         const uint64_t* eval_idx, int64_t eval_n, int eval_base, void* eval_out,
                         int num_sms, cudaStream_t st, bool* supported) {
  SmallArgs a{};
  a.net = net; a.pert = pert; a.prop = prop; a.cov = cov; a.res = res; a.ws = ws; a.n_base = n_base;
  a.bases = bases;
  a.eval_idx = eval_idx; a.eval_n = eval_n; a.eval_base = eval_base; a.eval_out = eval_out;
  *supported = true;
  const int L = net.L, n1 = net.sizes[1], n2 = net.sizes[2], n3 = L >= 3 ? net.sizes[3] : 0;
  // exact-width instantiations for the BASELINE's small net (25-10-5, configs 1 and 2): the
  // register arrays hold n_1 / n_2 values with no guarded padding iterations (the 16-wide form
  // spent ~60 % of cfg2's instructions on predicated-off iterations of the dense loops)
  if (L == 2 && n1 == 10 && n2 == 5) {
    if (net.numeric == MLPV_NUM_FP32) return run_small<MLPV_NUM_FP32, 2, 10, 5, 0>(a, num_sms, st);
    if (net.numeric == MLPV_NUM_Q4_12) return run_small<MLPV_NUM_Q4_12, 2, 10, 5, 0>(a, num_sms, st);
    if (net.numeric == MLPV_NUM_INT8) return run_small<MLPV_NUM_INT8, 2, 10, 5, 0>(a, num_sms, st);
  }
  if (L == 2 && n1 <= 16 && n2 <= 16) {
    if (net.numeric == MLPV_NUM_FP32) return run_small<MLPV_NUM_FP32, 2, 16, 16, 0>(a, num_sms, st);
    if (net.numeric == MLPV_NUM_Q4_12) return run_small<MLPV_NUM_Q4_12, 2, 16, 16, 0>(a, num_sms, st);
    if (net.numeric == MLPV_NUM_INT8) return run_small<MLPV_NUM_INT8, 2, 16, 16, 0>(a, num_sms, st);
  }
  if (L == 3 && n1 <= 16 && n2 <= 16 && n3 <= 16) {
    if (net.numeric == MLPV_NUM_FP32) return run_small<MLPV_NUM_FP32, 3, 16, 16, 16>(a, num_sms, st);
    if (net.numeric == MLPV_NUM_Q4_12) return run_small<MLPV_NUM_Q4_12, 3, 16, 16, 16>(a, num_sms, st);
    if (net.numeric == MLPV_NUM_INT8) return run_small<MLPV_NUM_INT8, 3, 16, 16, 16>(a, num_sms, st);
  }
  if (L == 3 && n1 <= 64 && n2 <= 32 && n3 <= 16 && net.numeric == MLPV_NUM_INT8)
    return run_small<MLPV_NUM_INT8, 3, 64, 32, 16>(a, num_sms, st);
  *supported = false;
  return cudaSuccess;
}

}  // namespace mlpv
