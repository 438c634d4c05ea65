// k_util.cu -- small device kernels around the check: result initialisation, merge of partial
// results (cross-GPU all-gather and resumed sub-ranges), neuron coverage
// and the float ambiguity widths tau (reading C20).
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "mlpv_internal.cuh"

namespace mlpv {

__global__ void k_init_result(DevResult r, int n_base, uint32_t n_words) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n_base) {
    r.checked[t] = 0; r.violated[t] = 0; r.flagged[t] = 0;
    r.first_cex[t] = kNone; r.first_cex_unflagged[t] = kNone;
  }
  for (uint32_t w = t; w < n_words; w += gridDim.x * blockDim.x) {
    if (r.cov_all) r.cov_all[w] = 0;
    if (r.cov_certain) r.cov_certain[w] = 0;
  }
}

// ---------------------------------------------------------------- restriction R on the Philox spaces
// (reading C27): one thread per candidate reconstructs the candidate
// pixel by pixel (readings C14/C15) and sums (x'_p - x_p)^2 in pixel order with separately rounded
// double operations (no contraction) -- the sum the definition states, so a candidate is inside R on
// the GPU iff it is by that definition -- or exactly in int64 for u8 (against floor(b^2 255^2)).
// One warp per 32 consecutive candidates of a base writes one mask word (ballot).
__device__ __forceinline__ uint4 philox_r(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return make_uint4(c0, c1, c2, c3);
}
// nearest bf16 value of v (8 significant bits, ties to even)
__device__ __forceinline__ double rne_bf16_d(double v) {
  if (v == 0.0) return v;
  int e;
  const double m = frexp(v, &e);
  return ldexp(rint(ldexp(m, 8)), e - 8);
}

__global__ void k_restrict_mask(DevNet net, const void* bases, DevPert p, uint32_t* mask, uint64_t len) {
  const int b = blockIdx.y;
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int n0 = net.sizes[0];
  bool in = false;
  if (i < len) {
    const uint64_t c = p.begin + i;
    const uint32_t k0 = (uint32_t)p.seed, k1 = (uint32_t)(p.seed >> 32);
    const bool u8 = net.numeric == MLPV_NUM_INT8;
    double s2 = 0.0;
    long long s2i = 0;
    for (int j = 0; j < (n0 + 31) / 32; j++) {
      const uint4 w = philox_r((uint32_t)c, (uint32_t)(c >> 32), (uint32_t)b, (uint32_t)j, k0, k1);
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      for (int q = 0; q < 32 && 32 * j + q < n0; q++) {
        const int px = 32 * j + q;
        const int l = (int)((ws[q >> 3] >> (4 * (q & 7))) & 15u);
        if (u8) {
          const int x = static_cast<const uint8_t*>(bases)[(size_t)b * n0 + px];
          const int y = max(0, min(255, x + l * p.step_i + p.origin_i));
          s2i += (long long)(y - x) * (y - x);
          continue;
        }
        const double x = (double)__uint_as_float((uint32_t)static_cast<const uint16_t*>(bases)[(size_t)b * n0 + px] << 16);
        double v;
        if (p.kind == MLPV_PERT_PHILOX_LATTICE) {
          const double off = rne_bf16_d(__dadd_rn(__dmul_rn((double)l, (double)p.step_f), (double)p.origin_f));
          v = __dadd_rn(x, off);
          v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
          v = rne_bf16_d(v);
        } else {
          v = __dadd_rn(x, __dadd_rn(p.origin_d, __dmul_rn((double)l, p.step_d)));
          if (p.kind == MLPV_PERT_PHILOX_CLAMP) v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        }
        const double d = __dadd_rn(v, -x);
        s2 = __dadd_rn(s2, __dmul_rn(d, d));
      }
    }
    in = u8 ? s2i <= p.r2_raw : s2 <= p.r2_f;
  }
  const uint32_t word = __ballot_sync(0xffffffffu, in);
  if ((threadIdx.x & 31) == 0 && i < len) mask[(size_t)b * p.rmask_wpb + (i >> 5)] = word;
}

cudaError_t launch_restrict_mask(const DevNet& net, const void* bases, int n_base, const DevPert& pert,
                                 uint32_t* mask, cudaStream_t st) {
  const uint64_t len = pert.end - pert.begin;
  if (len == 0) return cudaSuccess;
  dim3 grid((unsigned)((len + 127) / 128), (unsigned)n_base);
  k_restrict_mask<<<grid, 128, 0, st>>>(net, bases, pert, mask, len);
  return cudaGetLastError();
}

cudaError_t launch_init_result(const DevResult& r, int n_base, uint32_t n_words, cudaStream_t st) {
  const int n = n_base > (int)n_words ? n_base : (int)n_words;
  const int blocks = (n + 255) / 256 > 0 ? ((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024) : 1;
  k_init_result<<<blocks, 256, 0, st>>>(r, n_base, n_words);
  return cudaGetLastError();
}

__global__ void k_merge(MergeParts mp, int n_parts, int n_base, size_t n_words, DevResult out) {
  const DevResult* parts = mp.p;
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t b = t; b < (size_t)n_base; b += stride) {
    unsigned long long c = 0, v = 0, f = 0, x = kNone, xu = kNone;
    for (int p = 0; p < n_parts; p++) {
      c += parts[p].checked[b]; v += parts[p].violated[b]; f += parts[p].flagged[b];
      x = parts[p].first_cex[b] < x ? parts[p].first_cex[b] : x;
      xu = parts[p].first_cex_unflagged[b] < xu ? parts[p].first_cex_unflagged[b] : xu;
    }
    out.checked[b] = c; out.violated[b] = v; out.flagged[b] = f;
    out.first_cex[b] = x; out.first_cex_unflagged[b] = xu;
  }
  for (size_t w = t; w < n_words; w += stride) {
    uint32_t a = 0, ce = 0;
    for (int p = 0; p < n_parts; p++) {
      if (parts[p].cov_all) a |= parts[p].cov_all[w];
      if (parts[p].cov_certain) ce |= parts[p].cov_certain[w];
    }
    if (out.cov_all) out.cov_all[w] = a;
    if (out.cov_certain) out.cov_certain[w] = ce;
  }
}

cudaError_t launch_merge(const MergeParts& parts_dev, int n_parts, int n_base, size_t n_words,
                         const DevResult& out, cudaStream_t st) {
  const size_t n = (size_t)n_base > n_words ? (size_t)n_base : n_words;
  unsigned blocks = (unsigned)((n + 255) / 256);
  if (blocks < 1) blocks = 1;
  if (blocks > 1024) blocks = 1024;
  k_merge<<<blocks, 256, 0, st>>>(parts_dev, n_parts, n_base, n_words, out);
  return cudaGetLastError();
}

// One thread per (method, neuron).  Reading C9: neuron (l, i) is covered by method m iff it is
// an endpoint of a covered pair of m.
__global__ void k_neuron_cov(DevNet net, DevCov cov, const uint32_t* words, uint8_t* covered, uint32_t* counts) {
  const int T = net.trace_len;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 4 * T) return;
  const int m = t / T, g = t % T;
  int l = 1;
  while (l < net.L && g >= net.loff[l + 1]) l++;
  const int i = g - net.loff[l];
  bool cov_ = false;
  for (int p = 0; p < cov.n_pairs && !cov_; p++) {
    const int k = cov.lower[p], nk = net.sizes[k], nu = net.sizes[k + 1], wpr = (nu + 31) >> 5;
    const uint32_t o = cov.off[p][m];
    if (m < 2) {                                   // SS, SV: explicit pairs
      if (l == k) {
        for (int w = 0; w < wpr && !cov_; w++) cov_ = words[o + i * wpr + w] != 0;
      } else if (l == k + 1) {
        for (int r = 0; r < nk && !cov_; r++) cov_ = (words[o + r * wpr + (i >> 5)] >> (i & 31)) & 1;
      }
    } else {                                       // VS, VV: column masks
      if (l == k) {
        for (int w = 0; w < wpr && !cov_; w++) cov_ = words[o + w] != 0;
      } else if (l == k + 1) {
        cov_ = (words[o + (i >> 5)] >> (i & 31)) & 1;
      }
    }
  }
  covered[t] = cov_ ? 1 : 0;
  if (cov_) atomicAdd(&counts[m], 1u);
}

cudaError_t launch_neuron_cov(const DevNet& net, const DevCov& cov, const uint32_t* words,
                              uint8_t* covered, uint32_t* counts, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(counts, 0, 4 * sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  const int n = 4 * net.trace_len;
  k_neuron_cov<<<(n + 255) / 256, 256, 0, st>>>(net, cov, words, covered, counts);
  return cudaGetLastError();
}

// tau_l = 1e-6 + 1e-5 * max over bases of max |u_l^base| (float potentials), one block per layer
// tau_l = 1e-6 + 1e-5 max_b max_i |u_l^base| (reading C20): a grid of (layer, base chunk) blocks,
// max by atomicMax on the float bits (non-negative floats order as unsigned), then the affine map
__global__ void k_tau_max(DevNet net, const float* trace, int n_base, int per_blk, unsigned* mx) {
  const int l = blockIdx.y + 1;
  const int T = net.trace_len, n = net.sizes[l];
  const int b0 = blockIdx.x * per_blk, b1 = min(n_base, b0 + per_blk);
  float m = 0.f;
  for (int b = b0; b < b1; b++)
    for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmaxf(m, fabsf(trace[(size_t)b * T + net.loff[l] + i]));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&mx[l - 1], __float_as_uint(m));
}
__global__ void k_tau_final(int L, float* tau) {
  const int l = threadIdx.x;
  if (l < L) tau[l] = 1e-6f + 1e-5f * __uint_as_float(reinterpret_cast<unsigned*>(tau)[l]);
}

cudaError_t launch_tau(const DevNet& net, const void* trace, int n_base, float* tau_out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(tau_out, 0, sizeof(float) * net.L, st);
  if (e != cudaSuccess) return e;
  const int per_blk = 8;
  const dim3 grid((unsigned)((n_base + per_blk - 1) / per_blk), (unsigned)net.L);
  k_tau_max<<<grid, 256, 0, st>>>(net, static_cast<const float*>(trace), n_base, per_blk,
                                  reinterpret_cast<unsigned*>(tau_out));
  k_tau_final<<<1, 32, 0, st>>>(net.L, tau_out);
  return cudaGetLastError();
}

// Incremental bounds (NEXT-2): split the (step, index) keys of the check into step[b] (1-based,
// 0 = no counterexample in the ball) and the index.
__global__ void k_split_steps(DevResult r, int n_base, int32_t* step, int32_t* step_u) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_base) return;
  const unsigned long long m = (1ull << kStepShift) - 1;
  const unsigned long long k = r.first_cex[b], ku = r.first_cex_unflagged[b];
  step[b] = k == kNone ? 0 : (int32_t)(k >> kStepShift);
  step_u[b] = ku == kNone ? 0 : (int32_t)(ku >> kStepShift);
  if (k != kNone) r.first_cex[b] = k & m;
  if (ku != kNone) r.first_cex_unflagged[b] = ku & m;
}

cudaError_t launch_split_steps(const DevResult& r, int n_base, int32_t* step, int32_t* step_u, cudaStream_t st) {
  k_split_steps<<<(n_base + 127) / 128, 128, 0, st>>>(r, n_base, step, step_u);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ dataset-pair coverage (NEXT-3)
// The four covers of every unordered pair {x_a, x_b}, a < b, of an image set,
// OR-ed over all pairs (the set-level literals of PAPER.md:364-392 / 584-589).  Block a takes the
// pairs (a, b > a), one thread per b; words are OR-ed into a block copy in smem when it fits,
// then flushed.  Same predicates as the check's epilogue (k_small cover_pair) with x_a in the
// role of the base; fixed-point distances in int64 (exact).  Float: the pair's bits also go to
// the certain set unless a predicate it used lies within tau of its boundary (reading C20).
template <typename P, typename D>
__global__ void __launch_bounds__(128) k_pair_cov(DevNet net, DevCov cov, const P* trace, int n,
                                                  uint32_t* g_all, uint32_t* g_cert, int in_smem) {
  extern __shared__ uint32_t s_w[];
  constexpr bool FL = std::is_same<P, float>::value;
  const int a = blockIdx.x;
  uint32_t* wa = in_smem ? s_w : g_all;
  uint32_t* wc = in_smem ? s_w + cov.n_words : g_cert;
  if (in_smem) {
    for (uint32_t w = threadIdx.x; w < 2 * cov.n_words; w += blockDim.x) s_w[w] = 0;
    __syncthreads();
  }
  const int T = net.trace_len;
  const P* ta = trace + (size_t)a * T;
  for (int b = a + 1 + threadIdx.x; b < n; b += blockDim.x) {
    const P* tb = trace + (size_t)b * T;
    for (int p = 0; p < cov.n_pairs; p++) {
      const int k = cov.lower[p], nk = net.sizes[k], nu = net.sizes[k + 1];
      const P* la = ta + net.loff[k];
      const P* lb = tb + net.loff[k];
      const P* ua = ta + net.loff[k + 1];
      const P* ub = tb + net.loff[k + 1];
      D th, tg;
      float tl = 0.f, tu = 0.f;
      if constexpr (FL) {
        th = cov.th_f[k - 1]; tg = cov.tg_f[k];
        tl = cov.tau_dev ? cov.tau_dev[k - 1] : cov.tau[k - 1];
        tu = cov.tau_dev ? cov.tau_dev[k] : cov.tau[k];
      } else {
        th = cov.th_i[k - 1]; tg = cov.tg_i[k];
      }
      int nsc = 0, istar = -1;
      D linf = D(0);
      bool amb = false;
      for (int i = 0; i < nk; i++) {
        const P x = la[i], y = lb[i];
        if ((x >= P(0)) != (y >= P(0))) { if (istar < 0) istar = i; nsc++; }
        D d = D(y) - D(x);
        d = d < D(0) ? -d : d;
        linf = d > linf ? d : linf;
        if (FL && (fabsf((float)x) < tl || fabsf((float)y) < tl)) amb = true;
      }
      if (!(nsc == 1 || (nsc == 0 && linf >= th))) continue;
      if (FL && nsc == 0 && fabsf((float)(linf - th)) < tl) amb = true;
      if (FL && !amb) {
        for (int j = 0; j < nu && !amb; j++) {
          const P x = ua[j], y = ub[j];
          const float d = fabsf((float)y - (float)x);
          if (fabsf((float)x) < tu || fabsf((float)y) < tu || fabsf(d - (float)tg) < tu) amb = true;
        }
      }
      const int wpr = (nu + 31) >> 5;
      const uint32_t o_sc = nsc == 1 ? cov.off[p][0] + istar * wpr : cov.off[p][2];
      const uint32_t o_vc = nsc == 1 ? cov.off[p][1] + istar * wpr : cov.off[p][3];
      for (int w = 0; w < wpr; w++) {
        uint32_t scw = 0, vcw = 0;
        for (int jj = 0; jj < 32 && 32 * w + jj < nu; jj++) {
          const P x = ua[32 * w + jj], y = ub[32 * w + jj];
          const bool sc = (x >= P(0)) != (y >= P(0));
          D d = D(y) - D(x);
          d = d < D(0) ? -d : d;
          scw |= (uint32_t)sc << jj;
          vcw |= (uint32_t)(!sc && d >= tg) << jj;
        }
        if (scw) { atomicOr(&wa[o_sc + w], scw); if (!amb) atomicOr(&wc[o_sc + w], scw); }
        if (vcw) { atomicOr(&wa[o_vc + w], vcw); if (!amb) atomicOr(&wc[o_vc + w], vcw); }
      }
    }
  }
  if (in_smem) {
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < cov.n_words; w += blockDim.x) {
      if (s_w[w]) atomicOr(&g_all[w], s_w[w]);
      if (s_w[cov.n_words + w]) atomicOr(&g_cert[w], s_w[cov.n_words + w]);
    }
  }
}

cudaError_t launch_pair_cov(const DevNet& net, const DevCov& cov, const void* trace, int n,
                            uint32_t* cov_all, uint32_t* cov_cert, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(cov_all, 0, 4ull * cov.n_words, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(cov_cert, 0, 4ull * cov.n_words, st);
  if (e != cudaSuccess || n < 2 || cov.n_words == 0) return e;
  const size_t smem = 8ull * cov.n_words;
  const int in_smem = smem <= 48 * 1024;
  const unsigned grid = (unsigned)(n - 1);
  if (net.numeric == MLPV_NUM_FP32 || net.numeric == MLPV_NUM_BF16)
    k_pair_cov<float, float><<<grid, 128, in_smem ? smem : 0, st>>>(net, cov, static_cast<const float*>(trace), n,
                                                                      cov_all, cov_cert, in_smem);
  else
    k_pair_cov<int32_t, long long><<<grid, 128, in_smem ? smem : 0, st>>>(net, cov, static_cast<const int32_t*>(trace),
                                                                           n, cov_all, cov_cert, in_smem);
  return cudaGetLastError();
}

}  // namespace mlpv
