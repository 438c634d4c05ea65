// mlpv_internal.cuh -- internal types shared by the host library and the sm_100a kernels.
// Not part of the ABI (include/mlpv.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/mlpv.h"

namespace mlpv {

constexpr int kMaxL = MLPV_MAX_LAYERS;
constexpr int kMaxPairs = MLPV_MAX_LAYERS - 1;
constexpr uint64_t kNone = ~0ull;

// Device copy of the network (original row-major layouts) + derived parameters.
struct DevNet {
  int L;
  int sizes[kMaxL + 1];
  int numeric, act;
  const void* W[kMaxL];       // device, row-major n_l x n_{l-1}
  const void* b[kMaxL];       // device, float | int32
  int shift[kMaxL];           // INT8 requant shifts
  const int16_t* knots;       // device [129] (PL sigmoid) or nullptr
  int trace_len;              // n_1 + .. + n_L
  int loff[kMaxL + 1];        // offset of layer l (1-based) in a trace
};

// Per-call coverage description, thresholds already in potential units.
struct DevCov {
  int n_pairs;
  int lower[kMaxPairs];
  uint32_t off[kMaxPairs][4];  // word offsets of SS, SV, VS, VV
  float tg_f[kMaxL], th_f[kMaxL], tau[kMaxL];   // float numerics (per layer l-1)
  const float* tau_dev;                        // if set, tau is read from here (device, [L])
  int64_t tg_i[kMaxL], th_i[kMaxL];            // fixed numerics (accumulator units)
  float near_tie;
  uint32_t n_words;
};

struct DevProp {
  int kind, target;
  float V_f;
  int64_t V_i;
};

struct DevPert {
  int kind, tuple, n_pixels, n_levels;
  const int32_t* pixels;      // device [n_pixels]
  uint64_t begin, end;        // index range
  uint64_t seed;
  float step_f, origin_f;     // PHILOX (BF16 values) / PHILOX_BOX (fp32 of the doubles)
  double step_d, origin_d;    // PHILOX_BOX / PHILOX_CLAMP
  // PHILOX_CLAMP on k_fused3: A = d * 2^clamp_s in fp16, d = min(max(origin + l step, -x), 1 - x);
  // the offsets come from the fp16-subnormal levels l * 2^-24 as fma(l 2^-24, clamp_m, clamp_c)
  int clamp_s;                // scale exponent s
  uint32_t clamp_m2, clamp_c2;   // fp16x2 {step 2^(24+s), step 2^(24+s)} / {origin 2^s, origin 2^s}
  int step_i, origin_i;       // PHILOX (INT8)
  uint64_t q2;                // TUPLE: q^2
  // restriction R (reading C27): keep delta(I^d, I) <= b; subset / tuple spaces (k_small)
  int restrict_on;
  double r2_f;                // float: b^2
  long long r2_raw;           // fixed: floor(b^2 S^2), S = 4096 (Q4.12) / 255 (INT8)
  const void* levels;         // device copy of the levels (set by the plan; k_small's filter)
  // restriction R on the Philox spaces: bit (b, c - rmask_begin) of rmask (words [n_base][rmask_wpb])
  // is set iff candidate c of base b lies inside R (k_restrict_mask); nullptr = no restriction
  const uint32_t* rmask;
  uint64_t rmask_begin;
  uint32_t rmask_wpb;
  // incremental bounds b_1 < .. < b_n (NEXT-2, reading C28): a violation's first_cex key is
  // (step << kStepShift) | index, step = smallest i with distance^2 <= r2 of b_i
  int n_steps;                // 0 = off
  const double* step_r2_f;    // device [n_steps] b_i^2 (float numerics)
  const long long* step_r2_raw;  // device [n_steps] floor(b_i^2 S^2) (fixed point)
  // early-exit passes (mlpv_incremental.early_exit): this pass checks only the candidates of step
  // `shell` (b_(shell-1) < delta <= b_shell) of the base inputs whose unflagged key in `decided`
  // (the result's first_cex_unflagged) is not from an earlier step; 0 = off
  int shell;
  const unsigned long long* decided;
};
constexpr int kStepShift = 48;   // candidate indices < 2^48 in incremental mode
constexpr int kMaxSteps = 2048;

struct DevResult {
  uint64_t *checked, *violated, *flagged, *first_cex, *first_cex_unflagged;
  uint32_t *cov_all, *cov_certain;
};

// Per-base workspace produced by the base prologue (K0).
struct BaseWS {
  void* trace;                // [n_base x T] float | int32 potentials of the base image
  int32_t* cls;               // [n_base] base class
  void* delta;                // [n_base x S x q x n_1] layer-1 delta tables (subset/tuple spaces)
  int S;                      // slots per base: n_0 (TUPLE) or K (SUBSET)
  float* base1;               // PHILOX_BOX: [n_base x n_1] W1 x + b1 + origin W1 1 (fp64 sum, fp32);
                              // PHILOX_CLAMP: W1 x + b1
  uint4* clampc;              // PHILOX_CLAMP: [n_base][ceil(n_0 / 8)][2] fp16x2 words {-x 2^s} | {(1-x) 2^s}
                              // of 8 pixels (pairs in pixel order; 0 beyond n_0)
  uint32_t* status;           // handle's device status word (input errors found on the device)
};
// bits of the device status word (mlpv_sync reports them)
constexpr uint32_t kStatusClampBase = 1u;      // a PHILOX_CLAMP base pixel outside [0, 1] or not fp16-exact
constexpr uint32_t kStatusQ412Base = 2u;       // a Q4.12 base pixel outside [0, 4096]

// Launchers (kernels in k_small.cu / k_large.cu / k_util.cu)
cudaError_t launch_base_prologue(const DevNet& net, const void* bases, int n_base, const DevPert& pert,
                                 const void* levels_dev, BaseWS ws, cudaStream_t st);
cudaError_t launch_small(const DevNet& net, const void* bases, int n_base, const DevPert& pert,
                         const DevProp& prop, const DevCov& cov, const DevResult& res, BaseWS ws,
                         const uint64_t* eval_idx, int64_t eval_n, int eval_base, void* eval_out,
                         int num_sms, cudaStream_t st, bool* supported);
cudaError_t launch_warp3(const DevNet& net, int n_base, const DevPert& pert, const DevProp& prop, const DevCov& cov,
                         const DevResult& res, BaseWS ws, int num_sms, cudaStream_t st, bool* supported);
cudaError_t launch_tc3(const DevNet& net, const void* bases, int n_base, const DevPert& pert, const DevProp& prop,
                       const DevCov& cov, const DevResult& res, BaseWS ws, int num_sms, cudaStream_t st,
                       bool* supported);
cudaError_t launch_init_result(const DevResult& r, int n_base, uint32_t n_words, cudaStream_t st);
constexpr int kMaxParts = 64;
struct MergeParts { DevResult p[kMaxParts]; };
cudaError_t launch_merge(const MergeParts& parts, int n_parts, int n_base, size_t n_words,
                         const DevResult& out, cudaStream_t st);
cudaError_t launch_neuron_cov(const DevNet& net, const DevCov& cov, const uint32_t* words,
                              uint8_t* covered, uint32_t* counts, cudaStream_t st);
cudaError_t launch_tau(const DevNet& net, const void* trace, int n_base, float* tau_out, cudaStream_t st);
cudaError_t launch_split_steps(const DevResult& r, int n_base, int32_t* step, int32_t* step_u, cudaStream_t st);
cudaError_t launch_restrict_mask(const DevNet& net, const void* bases, int n_base, const DevPert& pert,
                                 uint32_t* mask, cudaStream_t st);
// inside R? (Philox spaces with a restriction; always true otherwise)
__device__ __forceinline__ bool in_restriction(const DevPert& p, int b, uint64_t c) {
  if (!p.rmask) return true;
  const uint64_t i = c - p.rmask_begin;
  return (p.rmask[(size_t)b * p.rmask_wpb + (i >> 5)] >> (i & 31)) & 1u;
}
cudaError_t launch_pair_cov(const DevNet& net, const DevCov& cov, const void* trace, int n,
                            uint32_t* cov_all, uint32_t* cov_cert, cudaStream_t st);

#ifdef __CUDACC__
// Philox4x32-10 (reading C15) for a fixed counter prefix (c0, c1, c2) = (candidate lo, hi, base) and a
// varying block counter c3 = j, round keys rk[2r], rk[2r+1] precomputed on the host.
// Everything that does not depend on j is hoisted out (computed once per generator row and tile):
// in round 0 both products and the c0 lane; in round 1 the c0 product and the c2 / c3 lanes; in
// round 2 the c2 product.  Per call 4 fewer IMAD.WIDE and 2 fewer LOP3 than the plain ten-round
// loop (philox() in k_fused3 / k_large); the output is identical.
struct PhiloxRow { uint32_t d, k2, e, f5, g4, h; };
__device__ __forceinline__ PhiloxRow philox_row(uint32_t c0, uint32_t c1, uint32_t c2, const uint32_t (&rk)[20]) {
  PhiloxRow p;
  const uint32_t hi0a = __umulhi(0xD2511F53u, c0), lo0a = 0xD2511F53u * c0;
  const uint32_t hi1a = __umulhi(0xCD9E8D57u, c2), lo1a = 0xCD9E8D57u * c2;
  const uint32_t s0 = hi1a ^ c1 ^ rk[0];                 // round 0: c0 lane (j-free), c2 lane = d ^ j
  p.d = hi0a ^ rk[1];
  p.k2 = lo1a ^ rk[2];                                   // round 1's c1 ^ key
  const uint32_t hi0b = __umulhi(0xD2511F53u, s0), lo0b = 0xD2511F53u * s0;
  p.e = hi0b ^ lo0a ^ rk[3];                             // round 1: c2 lane (j-free)
  const uint32_t f = lo0b;                               // round 1: c3 lane
  p.f5 = f ^ rk[5];
  p.g4 = __umulhi(0xCD9E8D57u, p.e) ^ rk[4];             // round 2: product of the c2 lane
  p.h = 0xCD9E8D57u * p.e;
  return p;
}
__device__ __forceinline__ uint4 philox_j(const PhiloxRow& p, uint32_t j, const uint32_t (&rk)[20]) {
  const uint32_t s2 = p.d ^ j;                           // round 0
  const uint32_t hi1b = __umulhi(0xCD9E8D57u, s2), lo1b = 0xCD9E8D57u * s2;
  const uint32_t t0 = hi1b ^ p.k2;                       // round 1 (c1 = lo1b, c2 = e, c3 = f)
  const uint32_t hi0c = __umulhi(0xD2511F53u, t0), lo0c = 0xD2511F53u * t0;
  uint32_t c0 = p.g4 ^ lo1b, c1 = p.h, c2 = hi0c ^ p.f5, c3 = lo0c;   // round 2
#pragma unroll
  for (int r = 3; r < 10; r++) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ rk[2 * r], n2 = hi0 ^ c3 ^ rk[2 * r + 1];
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return make_uint4(c0, c1, c2, c3);
}

#endif

}  // namespace mlpv
