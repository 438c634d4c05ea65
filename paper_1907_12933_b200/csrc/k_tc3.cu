// k_tc3.cu -- SURVEY.md's kernel K2 for the enumerated spaces of small int8 nets (BASELINE config 3:
// 784-64-32-10, SUBSET spaces): thread = candidate, every layer a
// tcgen05 kind::i8 MMA (u8 activations x s8 weights -> s32 in TMEM, exact), the CUDA cores doing
// only the decode and the epilogues.
//
// Layer 1 as a contraction over the changed pixels (reading C14 / SURVEY a4): a
// subset candidate differs from its base image only at the K pixels p_k of the subset, so
//     u1[i] = (u1_base[i] - sum_k W1[i, p_k] x[p_k]) + sum_k W1[i, p_k] x'_k = C1[i] + (A B^T)[c, i]
// with A[c, k] = x'_k of candidate c (u8, K <= 32 padded to one 32-byte MMA K step) and B[i, k] =
// W1[i, p_k] (s8): one M128 x N(n1) x K32 MMA per 128 candidates; C1 is formed per base input in
// int32 (exact: the same integers as the delta tables of k_small / k_warp3).  Layers 2 and 3 are
// the requantised activations (reading C18: y = min(255, max(0, (u + 2^(sh-1)) >> sh))) written by
// the epilogue threads as the next layer's A rows (32-byte K blocks, no-swizzle K-major layout),
// against W2 / W3 resident in shared memory.
//
// A CTA (one per SM, 512 threads) runs four independent warpgroups; warpgroup g owns TMEM columns
// [128 g, 128 g + 128) (layer 1 in the first 64, layer 2 in the next 32, layer 3 in the next 16)
// and its own A tiles, and walks its own contiguous range of 128-candidate tiles: decode -> MMA1 ->
// E1 -> MMA2 -> E2 -> MMA3 -> E3.  One elected thread of the warpgroup issues its MMAs and commits
// them to the warpgroup's mbarrier; the four warpgroups interleave on the SM's tensor pipe and
// issue slots.  Predicates, covers (C3-C8), argmax / property (C12) and counts as k_warp3.
#include <cuda_runtime.h>

#include <cstdint>

#include "mlpv_internal.cuh"
#include "tc_ptx.cuh"

namespace mlpv {
using namespace tc;
namespace t3 {

constexpr int kM = 128;                     // candidates per tile (TMEM lanes)
constexpr int kWG = 4;                      // warpgroups per CTA
constexpr int kMaxN1 = 64, kMaxN2 = 32, kMaxN3 = 16;
constexpr uint32_t kTileA = kM * 32;        // one 32-byte K block of 128 rows (4 KB)
#ifndef MLPV_T3_SLEEP
#define MLPV_T3_SLEEP 96
#endif
constexpr uint32_t kSleepNs = MLPV_T3_SLEEP;  // between polls of a warpgroup's MMA barrier

struct Args {
  DevNet net;
  DevPert pert;
  DevProp prop;
  DevCov cov;
  DevResult res;
  BaseWS ws;
  const uint8_t* bases;                     // [n_base][n0] u8
  int n1p, n2p, n3p;                        // MMA N of each layer (multiples of 16)
  uint64_t tiles_per_base, n_tiles;
};

// per-warpgroup shared memory
struct alignas(16) WgSmem {
  uint8_t a1[kTileA];                       // layer-1 A: x'_k of the K subset pixels
  uint8_t a2[2 * kTileA];                   // layer-2 A: h1 (K = 64 in two blocks)
  uint8_t a3[kTileA];                       // layer-3 A: h2 (K = 32)
  int32_t c1[kMaxN1];                       // C1 of the staged base input
  int32_t ub1[kMaxN1], ub2[kMaxN2], ub3[kMaxN3];   // base potentials
  int32_t xk[32];                           // the base's pixel values at the subset pixels
  uint64_t mb;                              // MMA completion (one commit per layer)
};
struct alignas(16) Smem {
  uint8_t w1[kMaxN1 * 32];                  // B of layer 1: W1[i, p_k] (s8), rows i, K = 32
  uint8_t w2[2][kMaxN2 * 32];               // B of layer 2: W2 (s8), two 32-byte K blocks
  uint8_t w3[kMaxN3 * 32];                  // B of layer 3: W3 (s8)
  WgSmem wg[kWG];
  int32_t b2[kMaxN2], b3[kMaxN3];
  int16_t lv[256];                          // the levels (replacement values / offsets)
  uint32_t cov[256];                        // the CTA's coverage words
  unsigned long long cnt[2], cex;
  uint32_t tbase;
};

// byte offset of (row, byte b < 32) of a 32-byte-row K-major no-swizzle tile (lbo 128, sbo 256):
// 8-row x 16-byte core matrices, the two 16-byte halves of a row in K-adjacent core matrices
__device__ __forceinline__ uint32_t off32(uint32_t row, uint32_t b) { return none16_off(row, b >> 1) + (b & 1u); }

__device__ __forceinline__ uint32_t pack_req(int32_t u0, int32_t u1, int32_t u2, int32_t u3, int32_t r, int sh) {
  uint32_t hi2, w4;                          // y = clamp((u + r) >> sh, 0, 255), four per word
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, 0;" : "=r"(hi2) : "r"((u3 + r) >> sh), "r"((u2 + r) >> sh));
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(w4) : "r"((u1 + r) >> sh), "r"((u0 + r) >> sh), "r"(hi2));
  return w4;
}

// 32 / 16 consecutive words of a shared-memory int32 array (broadcast loads: every lane the same)
__device__ __forceinline__ void words32(const int32_t* p, uint32_t (&w)[32]) {
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const int4 v = reinterpret_cast<const int4*>(p)[k];
    w[4 * k] = (uint32_t)v.x; w[4 * k + 1] = (uint32_t)v.y; w[4 * k + 2] = (uint32_t)v.z; w[4 * k + 3] = (uint32_t)v.w;
  }
}
__device__ __forceinline__ void words16(const int32_t* p, uint32_t (&w)[16]) {
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int4 v = reinterpret_cast<const int4*>(p)[k];
    w[4 * k] = (uint32_t)v.x; w[4 * k + 1] = (uint32_t)v.y; w[4 * k + 2] = (uint32_t)v.z; w[4 * k + 3] = (uint32_t)v.w;
  }
}

__global__ void __launch_bounds__(kWG * 128, 1) k_tc3(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = warp >> 2, q = warp & 3;
  const int r = 32 * q + lane;              // row of the tile = TMEM lane
  const int t = threadIdx.x;
  const DevNet& net = a.net;
  const int n0 = net.sizes[0], n1 = net.sizes[1], n2 = net.sizes[2], n3 = net.sizes[3];
  const int K = a.pert.n_pixels, nq = a.pert.n_levels;
  WgSmem& W = S.wg[g];

  // ---- CTA setup: resident B tiles (K-padding and rows beyond n_l zero), biases, TMEM
  for (int i = t; i < (int)(sizeof(S.w1) + sizeof(S.w2) + sizeof(S.w3)) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(S.w1)[i] = 0;
  for (int i = t; i < 256; i += blockDim.x) S.cov[i] = 0;
  if (t < 2) S.cnt[t] = 0;
  if (t == 0) S.cex = kNone;
  __syncthreads();
  {
    const int8_t* W1 = static_cast<const int8_t*>(net.W[0]);
    const int8_t* W2 = static_cast<const int8_t*>(net.W[1]);
    const int8_t* W3 = static_cast<const int8_t*>(net.W[2]);
    for (int e = t; e < n1 * K; e += blockDim.x) {
      const int i = e / K, k = e % K;
      S.w1[off32(i, k)] = (uint8_t)W1[(size_t)i * n0 + a.pert.pixels[k]];
    }
    for (int e = t; e < n2 * n1; e += blockDim.x) {
      const int i = e / n1, j = e % n1;
      S.w2[j >> 5][off32(i, j & 31)] = (uint8_t)W2[e];
    }
    for (int e = t; e < n3 * n2; e += blockDim.x) {
      const int i = e / n2, j = e % n2;
      S.w3[off32(i, j)] = (uint8_t)W3[e];
    }
    for (int i = t; i < kMaxN2; i += blockDim.x) S.b2[i] = i < n2 ? static_cast<const int32_t*>(net.b[1])[i] : 0;
    for (int i = t; i < kMaxN3; i += blockDim.x) S.b3[i] = i < n3 ? static_cast<const int32_t*>(net.b[2])[i] : 0;
    for (int i = t; i < nq; i += blockDim.x) S.lv[i] = static_cast<const int16_t*>(a.pert.levels)[i];
    // A1 rows: the bytes k >= K stay zero (each tile writes only its K pixel bytes)
    for (int i = t; i < kWG * (int)kTileA / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(S.wg[i / (kTileA / 4)].a1)[i % (kTileA / 4)] = 0;
    if (q == 0 && lane == 0) { mbar_init(&W.mb, 1); }
  }
  if (warp == 0) { tmem_alloc(&S.tbase, 512); tmem_relinquish(); }
  fence_mbar_init();
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t D1 = S.tbase + 128u * g, D2 = D1 + 64u, D3 = D1 + 96u;
  const uint32_t loff = (uint32_t)(32 * q) << 16;

  const int sh1 = net.shift[0], sh2 = net.shift[1];
  const int32_t r1 = sh1 > 0 ? (1 << (sh1 - 1)) : 0, r2 = sh2 > 0 ? (1 << (sh2 - 1)) : 0;
  const uint32_t m1a = n1 >= 32 ? 0xFFFFFFFFu : ((1u << n1) - 1u);
  const uint32_t m1b = n1 >= 64 ? 0xFFFFFFFFu : (n1 > 32 ? ((1u << (n1 - 32)) - 1u) : 0u);
  const uint32_t m2 = n2 >= 32 ? 0xFFFFFFFFu : ((1u << n2) - 1u), m3 = (1u << n3) - 1u;
  int p12 = -1, p23 = -1;
  for (int p = 0; p < a.cov.n_pairs; p++) {
    if (a.cov.lower[p] == 1) p12 = p;
    if (a.cov.lower[p] == 2) p23 = p;
  }
  const int32_t tg2 = (int32_t)a.cov.tg_i[1], tg3 = (int32_t)a.cov.tg_i[2];
  const int32_t th1 = (int32_t)a.cov.th_i[0], th2 = (int32_t)a.cov.th_i[1];
  const int pkind = a.prop.kind, ptarget = a.prop.target;
  const int32_t pV = (int32_t)a.prop.V_i;
  const uint32_t id1 = idesc_i8(kM, (uint32_t)a.n1p, 0, 1), id2 = idesc_i8(kM, (uint32_t)a.n2p, 0, 1),
                 id3 = idesc_i8(kM, (uint32_t)a.n3p, 0, 1);
  const bool issuer = q == 0 && lane == 0;
  const int T = net.trace_len;
  const bool offs = a.pert.kind == MLPV_PERT_SUBSET_OFFSET;
  const bool pow2 = (nq & (nq - 1)) == 0;
  const int qb = __ffs(nq) - 1;

  // this warpgroup's contiguous tile range
  const uint64_t G = (uint64_t)gridDim.x * kWG, gi = (uint64_t)blockIdx.x * kWG + g;
  const uint64_t t0 = a.n_tiles * gi / G, t1 = a.n_tiles * (gi + 1) / G;
  uint32_t mph = 0;                          // parity of W.mb's next phase
  int cur_b = -1;
  uint32_t nb1a = 0, nb1b = 0, nb2 = 0, nb3 = 0;
  int base_cls = 0;
  unsigned long long my_chk = 0, my_v = 0, my_cex = kNone;
  auto wg_bar = [&]() { named_bar(1 + g, 128); };
  // counts and first counterexample of base input bb, reduced over the warp (bb is warp-uniform:
  // the whole warpgroup works on one tile at a time)
  auto flush = [&](int bb) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      my_chk += __shfl_xor_sync(0xffffffffu, my_chk, o);
      my_v += __shfl_xor_sync(0xffffffffu, my_v, o);
      const unsigned long long x = __shfl_xor_sync(0xffffffffu, my_cex, o);
      my_cex = x < my_cex ? x : my_cex;
    }
    if (lane == 0 && bb >= 0) {
      if (my_chk) atomicAdd(reinterpret_cast<unsigned long long*>(&a.res.checked[bb]), my_chk);
      if (my_v) atomicAdd(reinterpret_cast<unsigned long long*>(&a.res.violated[bb]), my_v);
      if (my_cex != kNone) {
        atomicMin(reinterpret_cast<unsigned long long*>(&a.res.first_cex[bb]), my_cex);
        atomicMin(reinterpret_cast<unsigned long long*>(&a.res.first_cex_unflagged[bb]), my_cex);
      }
    }
    my_chk = 0; my_v = 0; my_cex = kNone;
  };
  auto wait_mma = [&]() {
    if (lane == 0) mbar_wait_sleep(&W.mb, mph, kSleepNs);
    __syncwarp();
    mph ^= 1u;
    fence_after();
  };

  // (base input and tile offset advanced incrementally: no 64-bit division per tile)
  int tb = (int)(t0 / a.tiles_per_base);
  uint64_t toff = t0 % a.tiles_per_base;
  for (uint64_t tl = t0; tl < t1; tl++, toff++) {
    if (toff == a.tiles_per_base) { toff = 0; tb++; }
    const int b = tb;
    const uint64_t start = a.pert.begin + toff * kM;
    const uint64_t rem = a.pert.end - start;
    const int nvalid = rem < (uint64_t)kM ? (int)rem : kM;
    const bool valid = r < nvalid;
    const uint8_t* xb = a.bases + (size_t)b * n0;
    if (b != cur_b) {
      flush(cur_b);
      // ---- stage the base input: C1 = u1_base - sum_k W1[:, p_k] x[p_k], base potentials
      wg_bar();                              // the previous base's values are no longer read
      const int32_t* tr = static_cast<const int32_t*>(a.ws.trace) + (size_t)b * T;
      if (r < kMaxN1) {
        int32_t c = 0, u = 0;
        if (r < n1) {
          u = tr[net.loff[1] + r];
          c = u;
          const int8_t* W1 = static_cast<const int8_t*>(net.W[0]) + (size_t)r * n0;
          for (int k = 0; k < K; k++) {
            const int p = a.pert.pixels[k];
            c -= (int32_t)W1[p] * (int32_t)xb[p];
          }
        }
        W.c1[r] = c;
        W.ub1[r] = u;
      }
      if (r < kMaxN2) W.ub2[r] = r < n2 ? tr[net.loff[2] + r] : 0;
      if (r < 32) W.xk[r] = r < K ? (int32_t)xb[a.pert.pixels[r]] : 0;
      if (r < kMaxN3) W.ub3[r] = r < n3 ? tr[net.loff[3] + r] : 0;
      wg_bar();
      nb1a = nb1b = nb2 = nb3 = 0;
      for (int i = 0; i < 32; i++) {
        nb1a |= (uint32_t)(W.ub1[i] < 0) << i;
        nb1b |= (uint32_t)(W.ub1[32 + i] < 0) << i;
        nb2 |= (uint32_t)(W.ub2[i] < 0) << i;
      }
      for (int i = 0; i < kMaxN3; i++) nb3 |= (uint32_t)(W.ub3[i] < 0) << i;
      nb1a &= m1a; nb1b &= m1b; nb2 &= m2; nb3 &= m3;
      base_cls = a.ws.cls[b];
      cur_b = b;
    }
    const uint64_t c = start + (uint64_t)r;

    // ---- decode (reading C14: mixed radix, the last pixel the least significant digit) -> A1 row:
    // one byte per subset pixel (x'_k: the replacement value, or the clamped offset pixel)
    {
      const uint64_t cv = valid ? c : a.pert.begin;
      // off32(r, k) = rowbase(r) + (k >> 4) * 128 + (k & 15)
      uint8_t* arow = W.a1 + ((uint32_t)(r >> 3) * 256u + (uint32_t)(r & 7) * 16u);
      auto put = [&](int k, int d) {
        int v = S.lv[d];
        if (offs) v = max(0, min(255, W.xk[k] + v));
        arow[(k >> 4) * 128 + (k & 15)] = (uint8_t)v;
      };
      if (pow2) {
        uint64_t cc = cv;
        for (int k = K - 1; k >= 0; k--) { put(k, (int)(cc & (uint64_t)(nq - 1))); cc >>= qb; }
      } else if (a.pert.end <= (1ull << 32)) {
        uint32_t cc = (uint32_t)cv;
        for (int k = K - 1; k >= 0; k--) { put(k, (int)(cc % (uint32_t)nq)); cc /= (uint32_t)nq; }
      } else {
        uint64_t cc = cv;
        for (int k = K - 1; k >= 0; k--) { put(k, (int)(cc % (uint64_t)nq)); cc /= (uint64_t)nq; }
      }
    }
    // the accumulators start from the offsets (C1, b2, b3 written into TMEM by tcgen05.st, the MMAs
    // accumulate onto them): no per-neuron adds in the epilogues
    {
      uint32_t cw[32];
      words32(W.c1, cw);
      tmem_st32(D1 + loff, cw);
      if (a.n1p > 32) {
        words32(W.c1 + 32, cw);
        tmem_st32(D1 + loff + 32u, cw);
      }
      tmem_st_wait();
    }
    fence_proxy_async();
    fence_before();
    wg_bar();
    if (issuer) {
      fence_after();
      mma_i8_ss(D1, sdesc_none(smem_u32(W.a1), 128, 256), sdesc_none(smem_u32(S.w1), 128, 256), id1, 1u);
      mma_commit(&W.mb);
    }
    wait_mma();

    // ---- E1: u1 = C1 + acc (C1 preloaded), sign changes, requantised h1 -> A2 rows
    int32_t u1[64];
    {
      uint32_t v[32];
      tmem_ld32(D1 + loff, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i++) u1[i] = (int32_t)v[i];
      if (a.n1p > 32) {
        tmem_ld32(D1 + loff + 32u, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i++) u1[32 + i] = (int32_t)v[i];
      } else {
#pragma unroll
        for (int i = 0; i < 32; i++) u1[32 + i] = 0;
      }
      if (a.n1p == 48) {                     // columns 48..63 are not this layer's
#pragma unroll
        for (int i = 48; i < 64; i++) u1[i] = 0;
      } else if (a.n1p == 16) {
#pragma unroll
        for (int i = 16; i < 32; i++) u1[i] = 0;
      }
    }
    uint32_t ng1a = 0, ng1b = 0;
#pragma unroll
    for (int i = 31; i >= 0; i--) {
      ng1a = __funnelshift_l((uint32_t)u1[i], ng1a, 1);
      ng1b = __funnelshift_l((uint32_t)u1[32 + i], ng1b, 1);
    }
    const uint32_t sc1a = (ng1a & m1a) ^ nb1a, sc1b = (ng1b & m1b) ^ nb1b;
    const int nsc1 = __popc(sc1a) + __popc(sc1b);
    {
      uint32_t hw[16];
#pragma unroll
      for (int k = 0; k < 16; k++) hw[k] = pack_req(u1[4 * k], u1[4 * k + 1], u1[4 * k + 2], u1[4 * k + 3], r1, sh1);
      // padded neurons (n1 <= i < 64) hold u = 0 -> h = 0; W2's matching K columns are zero
#pragma unroll
      for (int kb = 0; kb < 2; kb++) {
        *reinterpret_cast<uint4*>(W.a2 + kb * kTileA + off32(r, 0)) = make_uint4(hw[8 * kb], hw[8 * kb + 1], hw[8 * kb + 2], hw[8 * kb + 3]);
        *reinterpret_cast<uint4*>(W.a2 + kb * kTileA + off32(r, 16)) = make_uint4(hw[8 * kb + 4], hw[8 * kb + 5], hw[8 * kb + 6], hw[8 * kb + 7]);
      }
    }
    // pair (1, 2) condition: one layer-1 sign change, or none and an L-inf change >= th1 (C3-C8)
    bool cond1 = false;
    if (p12 >= 0 && valid && nsc1 <= 1) {
      cond1 = nsc1 == 1;
      if (!cond1) {
        int32_t d = 0;
#pragma unroll
        // (neurons >= n1 hold u = ub = 0)
        const int4* ub4 = reinterpret_cast<const int4*>(W.ub1);
#pragma unroll
        for (int k = 0; k < 16; k++) {
          const int4 bv = ub4[k];
          d = max(d, max(max(abs(u1[4 * k] - bv.x), abs(u1[4 * k + 1] - bv.y)), max(abs(u1[4 * k + 2] - bv.z), abs(u1[4 * k + 3] - bv.w))));
        }
        cond1 = d >= th1;
      }
    }
    const int istar1 = sc1a ? __ffs(sc1a) - 1 : (sc1b ? 32 + __ffs(sc1b) - 1 : -1);
    {
      uint32_t bw[32];
      words32(S.b2, bw);
      tmem_st32(D2 + loff, bw);
      tmem_st_wait();
    }
    fence_proxy_async();
    fence_before();
    wg_bar();
    if (issuer) {
      fence_after();
      mma_i8_ss(D2, sdesc_none(smem_u32(W.a2), 128, 256), sdesc_none(smem_u32(S.w2[0]), 128, 256), id2, 1u);
      if (a.n1p > 32)
        mma_i8_ss(D2, sdesc_none(smem_u32(W.a2 + kTileA), 128, 256), sdesc_none(smem_u32(S.w2[1]), 128, 256), id2, 1u);
      mma_commit(&W.mb);
    }
    wait_mma();

    // ---- E2: u2 = b2 + acc, sign changes, h2 -> A3 rows, pair (1, 2) covers
    int32_t u2[32];
    {
      uint32_t v[32];
      tmem_ld32(D2 + loff, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i++) u2[i] = (int32_t)v[i];
    }
    // (N = n2p columns were computed; columns >= n2p of the ld are not ours: mask them out)
#pragma unroll
    if (a.n2p == 16) {                       // columns 16..31 are not this layer's
#pragma unroll
      for (int i = 16; i < 32; i++) u2[i] = 0;
    }
    uint32_t ng2 = 0;
#pragma unroll
    for (int i = 31; i >= 0; i--) ng2 = __funnelshift_l((uint32_t)u2[i], ng2, 1);
    const uint32_t sc2 = (ng2 & m2) ^ nb2;
    const int nsc2 = __popc(sc2);
    {
      uint32_t hw[8];
#pragma unroll
      for (int k = 0; k < 8; k++) hw[k] = pack_req(u2[4 * k], u2[4 * k + 1], u2[4 * k + 2], u2[4 * k + 3], r2, sh2);
      *reinterpret_cast<uint4*>(W.a3 + off32(r, 0)) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      *reinterpret_cast<uint4*>(W.a3 + off32(r, 16)) = make_uint4(hw[4], hw[5], hw[6], hw[7]);
    }
    if (cond1) {
      uint32_t vc2 = 0;
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const int4 bv = reinterpret_cast<const int4*>(W.ub2)[k];
        vc2 |= ((uint32_t)(abs(u2[4 * k] - bv.x) >= tg2) | ((uint32_t)(abs(u2[4 * k + 1] - bv.y) >= tg2) << 1) |
                ((uint32_t)(abs(u2[4 * k + 2] - bv.z) >= tg2) << 2) | ((uint32_t)(abs(u2[4 * k + 3] - bv.w) >= tg2) << 3)) << (4 * k);
      }
      vc2 &= ~sc2 & m2;
      const uint32_t* off = a.cov.off[p12];
      const uint32_t is = nsc1 == 1 ? off[0] + istar1 : off[2], iv = nsc1 == 1 ? off[1] + istar1 : off[3];
      if (sc2 && (S.cov[is] & sc2) != sc2) atomicOr(&S.cov[is], sc2);
      if (vc2 && (S.cov[iv] & vc2) != vc2) atomicOr(&S.cov[iv], vc2);
    }
    bool cond2 = false;
    if (p23 >= 0 && valid && nsc2 <= 1) {
      cond2 = nsc2 == 1;
      if (!cond2) {
        int32_t d = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
          const int4 bv = reinterpret_cast<const int4*>(W.ub2)[k];
          d = max(d, max(max(abs(u2[4 * k] - bv.x), abs(u2[4 * k + 1] - bv.y)), max(abs(u2[4 * k + 2] - bv.z), abs(u2[4 * k + 3] - bv.w))));
        }
        cond2 = d >= th2;
      }
    }
    {
      uint32_t bw[16];
      words16(S.b3, bw);
      tmem_st16(D3 + loff, bw);
      tmem_st_wait();
    }
    fence_proxy_async();
    fence_before();
    wg_bar();
    if (issuer) {
      fence_after();
      mma_i8_ss(D3, sdesc_none(smem_u32(W.a3), 128, 256), sdesc_none(smem_u32(S.w3), 128, 256), id3, 1u);
      mma_commit(&W.mb);
    }
    wait_mma();

    // ---- E3: logits, argmax (lowest index on ties), property (C12), pair (2, 3) covers, counts
    int32_t y[16];
    {
      uint32_t v[16];
      tmem_ld16(D3 + loff, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; i++) y[i] = (int32_t)v[i];
    }
    fence_before();                          // E3's TMEM reads precede the next tile's MMAs
    int cls = 0;
    int32_t top = y[0];
#pragma unroll
    for (int i = 1; i < 16; i++) if (i < n3 && y[i] > top) { top = y[i]; cls = i; }
    bool viol;
    if (pkind == MLPV_PROP_THRESHOLD_LITERAL || pkind == MLPV_PROP_THRESHOLD_LITERAL_ALL) {
      const int D = ptarget >= 0 ? ptarget : base_cls;
      bool any = false, all = true;
      int32_t yD = 0;
#pragma unroll
      for (int i = 0; i < 16; i++)
        if (i < n3) {
          if (i == D) yD = y[i];
          if (i != D && y[i] > pV) any = true;
          if (i != D && !(y[i] > pV)) all = false;
        }
      viol = yD < pV && (pkind == MLPV_PROP_THRESHOLD_LITERAL_ALL ? all : any);
    } else {
      viol = pkind == MLPV_PROP_TARGET_NEVER ? cls == ptarget : cls != base_cls;
    }
    viol = viol && valid;
    if (cond2) {
      uint32_t ng3 = 0, vc3 = 0;
#pragma unroll
      for (int i = 0; i < 16; i++) {
        ng3 |= (uint32_t)(y[i] < 0) << i;
        vc3 |= (uint32_t)(abs(y[i] - W.ub3[i]) >= tg3) << i;
      }
      const uint32_t sc3 = (ng3 & m3) ^ nb3;
      vc3 &= ~sc3 & m3;
      const uint32_t* off = a.cov.off[p23];
      const int istar2 = sc2 ? __ffs(sc2) - 1 : 0;
      const uint32_t is = nsc2 == 1 ? off[0] + istar2 : off[2], iv = nsc2 == 1 ? off[1] + istar2 : off[3];
      if (sc3 && (S.cov[is] & sc3) != sc3) atomicOr(&S.cov[is], sc3);
      if (vc3 && (S.cov[iv] & vc3) != vc3) atomicOr(&S.cov[iv], vc3);
    }
    if (valid) my_chk++;
    if (viol) { my_v++; if (c < my_cex) my_cex = c; }
  }

  // ---- a9: counts of the last base input, then the CTA's coverage words
  flush(cur_b);
  fence_before();
  __syncthreads();
  for (uint32_t w = t; w < a.cov.n_words; w += blockDim.x)
    if (S.cov[w]) { atomicOr(&a.res.cov_all[w], S.cov[w]); atomicOr(&a.res.cov_certain[w], S.cov[w]); }
  if (warp == 0) tmem_dealloc(S.tbase, 512);
}

}  // namespace t3

// the tensor-core kernel when it applies (int8, 3 layers, n1 <= 64, n2 <= 32, n3 <= 16, subset
// spaces with K <= 32 pixels, a plain check); *supported = false otherwise
cudaError_t launch_tc3(const DevNet& net, const void* bases, int n_base, const DevPert& pert, const DevProp& prop,
                       const DevCov& cov, const DevResult& res, BaseWS ws, int num_sms, cudaStream_t st,
                       bool* supported) {
  *supported = net.numeric == MLPV_NUM_INT8 && net.L == 3 && net.sizes[1] <= t3::kMaxN1 &&
               net.sizes[2] <= t3::kMaxN2 && net.sizes[3] <= t3::kMaxN3 &&
               (pert.kind == MLPV_PERT_SUBSET_REPLACE || pert.kind == MLPV_PERT_SUBSET_OFFSET) &&
               !pert.restrict_on && pert.n_steps == 0 && pert.n_pixels >= 1 && pert.n_pixels <= 32 &&
               cov.n_words <= 256 && pert.levels != nullptr && pert.pixels != nullptr;
  if (!*supported) return cudaSuccess;
  t3::Args a;
  a.net = net; a.pert = pert; a.prop = prop; a.cov = cov; a.res = res; a.ws = ws;
  a.bases = static_cast<const uint8_t*>(bases);
  auto p16 = [](int n) { return (n + 15) / 16 * 16; };
  a.n1p = p16(net.sizes[1]); a.n2p = p16(net.sizes[2]); a.n3p = p16(net.sizes[3]);
  const uint64_t len = pert.end - pert.begin;
  a.tiles_per_base = (len + t3::kM - 1) / t3::kM;
  a.n_tiles = a.tiles_per_base * (uint64_t)n_base;
  if (a.n_tiles == 0) return cudaSuccess;
  const size_t smem = sizeof(t3::Smem) + 1024;
  cudaError_t e = cudaFuncSetAttribute(t3::k_tc3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  uint64_t grid = (uint64_t)num_sms;
  const uint64_t need = (a.n_tiles + t3::kWG - 1) / t3::kWG;
  if (grid > need) grid = need;
  t3::k_tc3<<<(unsigned)grid, t3::kWG * 128, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace mlpv
