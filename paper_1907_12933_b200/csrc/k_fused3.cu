// k_fused3.cu -- the specialised large-net kernel for 3-layer bf16 nets with 256-wide hidden layers
// (BASELINE config 4: 784-256-256-10).  Everything stays on chip:
//
//   * a CTA pair (cluster of 2, tcgen05.mma.cta_group::2, M = 256 candidates) shares each weight
//     tile: every CTA loads only its half (128 of the 256 output neurons), halving L2->SM traffic
//     and shared-memory bandwidth per MMA;
//   * layer 1: A = Philox-lattice candidates written by 4 generator warps into a SWIZZLE_128B ring,
//     B = W1 half tiles streamed by cp.async.bulk; the layer bias rides along as three extra K
//     columns (bf16 hi/mid/lo of the fp32 bias) in the otherwise zero K padding (784 -> 832);
//   * the layer-1 accumulator (TMEM columns 0-255) is turned in place by the epilogue into the
//     fp16 hi/lo split of the hidden activations (reading C19), which is the A operand of layer 2
//     straight from TMEM (tcgen05.mma ... [a_tmem]); layer 2 accumulates in columns 256-511;
//   * layer 3 (N = 10, padded to 32): the epilogue stages 32-neuron chunks of [hi | lo] in shared
//     memory and a second issuer thread runs the small MMAs into the drained columns 256-287;
//   * 8 epilogue warps (two groups of four, one thread per candidate row) evaluate the predicates
//     and coverage with the sign / L-inf / min|u| summaries of each
//     32-neuron piece, and only rare candidates take the per-neuron coverage path.
//
// Warp roles (15 warps): 0 producer, 1 MMA issuer (leader) / relay (peer) and TMEM owner,
// 2 layer-3 issuer (leader), 3-6 generator, 7-14 epilogue (two groups of four warps covering the
// four TMEM lane quadrants each).  The leader (cluster rank 0) issues every MMA;
// the peer signals its readiness by remote mbarrier arrives; MMA completion is committed with
// multicast to both CTAs.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "mlpv_internal.cuh"
#include "tc_ptx.cuh"

namespace mlpv {
using namespace tc;

namespace f3 {
#ifdef MLPV_TRACE
// debug timeline (tools/trace_fused3.py): clock64 stamps of the first 64 tiles of cluster 0
__device__ unsigned long long g_trace[2][64][32];
#define TR(tl, ev) do { if (cluster == 0 && (tl) < 64) g_trace[rank][(tl)][(ev)] = clock64(); } while (0)
#else
#define TR(tl, ev) do { } while (0)
#endif
constexpr int kThreads = 480;
constexpr int kSG = 3;                       // generator ring stages
constexpr int kSW = 4;                       // weight ring stages
constexpr uint32_t kTile = 16384;            // 128 rows x 128 B
constexpr int kN1 = 256, kN2 = 256, kN3P = 32;
constexpr int kNkb2 = kN1 / 64;              // W2 K blocks (64 fp16 per 128-B row)
constexpr int kChunks = kN2 / 32;            // layer-3 chunks (32 neurons of layer 2)
constexpr uint32_t kW3Chunk = 16u * 128u;    // per CTA: 16 rows x 128 B
constexpr int kMaxN0 = 1024;

struct Args {
  int n0, n3, nkb1;
  uint64_t n_pairs_tiles;                    // pair tiles (256 candidates each)
  uint64_t tiles_per_base;
  const uint8_t* wstream;                    // [rank][nkb1 + 4][16 KB] W1 (with bias columns) then W2 (fp16)
  const uint8_t* w3;                         // [rank][kChunks][2 KB]
  const float* b2;                           // [256]
  const float* b3;                           // [n3]
  const uint16_t* bases;                     // [n_base][n0] bf16
  DevPert pert;
  DevProp prop;
  DevCov cov;
  DevResult res;
  const float* trace;                        // base potentials [n_base][T]
  const int32_t* cls;                        // base classes
  int T;
  int pair12, pair23;                        // coverage pair indices or -1
  const uint64_t* eval_idx;
  int64_t eval_n;
  int eval_base;
  float* eval_out;
};

struct alignas(16) Smem {                    // (dynamic part follows the 1 KiB-aligned tiles)
  uint64_t g_full[kSG], g_empty[kSG], w_full[kSW], w_empty[kSW];
  uint64_t acc1_full, acc2_full, acc3_full, h1_ready, acc2_free;
  uint64_t h2c_full[4], h2c_empty[4];
  uint32_t tbase;
  int base_g, base_e;                        // base input whose data is staged (generator / epilogue)
  alignas(16) float ub1[kN1];
  alignas(16) float ub2[kN2];
  alignas(16) float ub3[kN3P];
  alignas(16) float b2[kN2];
  alignas(16) float b3[kN3P];
  uint32_t nb1[8], nb2[8], nb3;
  float minub[3];
  // per-candidate summaries exchanged between the two epilogue groups
  int x_nsc[2][128], x_first[2][128];
  uint32_t x_fw[2][128];
  float x_linf[2][128], x_minab[2][128], x_vcamb[2][128];
  alignas(16) uint16_t xg[kMaxN0 + 128];     // base image (bf16) for the generator, zero padded
};

constexpr size_t kTilesBytes = (size_t)kSG * kTile + (size_t)kSW * kTile + (size_t)kChunks * kW3Chunk + 4 * (size_t)kTile;
constexpr size_t kSmemBytes = 1024 + kTilesBytes + sizeof(Smem);

struct TileInfo {
  int b;
  uint64_t start;     // first candidate index of the pair tile (range mode) or list position (eval)
  int nvalid;         // valid rows of the pair tile (0..256)
};

__device__ __forceinline__ TileInfo tile_info(const Args& a, uint64_t t) {
  TileInfo ti;
  if (a.eval_idx) {
    ti.b = a.eval_base;
    ti.start = t * 256;
    const int64_t rem = a.eval_n - (int64_t)ti.start;
    ti.nvalid = rem < 256 ? (int)rem : 256;
  } else {
    ti.b = (int)(t / a.tiles_per_base);
    ti.start = a.pert.begin + (t % a.tiles_per_base) * 256;
    const uint64_t rem = a.pert.end - ti.start;
    ti.nvalid = rem < 256 ? (int)rem : 256;
  }
  return ti;
}

__device__ __forceinline__ uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
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

__device__ __forceinline__ uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t hfma2_relu(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.relu.bf16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t hmin2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("min.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hsub2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// 4 lattice pixel pairs from one Philox word (nibble n -> pixel n), x2[k] = base pixels (bf16x2).
// x' = min(relu(RNE(x + RNE(l*step + origin))), 1)  (reading C14)
__device__ __forceinline__ uint4 lattice_word(uint32_t w, uint4 x2, uint32_t step2, uint32_t org2) {
  const uint32_t lo = w & 0x0F0F0F0Fu, hi = (w >> 4) & 0x0F0F0F0Fu;
  const uint32_t one2 = 0x3F803F80u, c128 = 0x43004300u;
  uint32_t o[4];
  const uint32_t xs[4] = {x2.x, x2.y, x2.z, x2.w};
#pragma unroll
  for (int k = 0; k < 4; k++) {
    // bytes [lo_k, -, hi_k, -] -> bf16x2 (128 + la, 128 + lb): one PRMT + one LOP3
    const uint32_t sel = (uint32_t)k * 0x11u + (4u + (uint32_t)k) * 0x1100u;
    const uint32_t pair = (__byte_perm(lo, hi, sel) & 0x00FF00FFu) | c128;
    const uint32_t l = hsub2(pair, c128);                 // exact: (la, lb)
    const uint32_t off = hfma2(l, step2, org2);           // RNE(l*step + origin)
    o[k] = hmin2(hfma2_relu(xs[k], one2, off), one2);     // min(relu(RNE(x + off)), 1)
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

__device__ __forceinline__ uint32_t f2h2_rz_relu(float lo, float hi) {
  uint32_t d;
  asm("cvt.rz.relu.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
__device__ __forceinline__ uint32_t f2h2_rn_relu(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
// h = max(u, 0) = hi + lo + O(2^-21 h):  hi = RZ_f16(h), lo = RN_f16(h - hi)  (both relu'd)
__device__ __forceinline__ void split_pair(float u0, float u1, uint32_t& hi2, uint32_t& lo2) {
  hi2 = f2h2_rz_relu(u0, u1);
  const float h0 = __half2float(__ushort_as_half((unsigned short)(hi2 & 0xFFFFu)));
  const float h1 = __half2float(__ushort_as_half((unsigned short)(hi2 >> 16)));
  lo2 = f2h2_rn_relu(u0 - h0, u1 - h1);
}

__device__ __forceinline__ void arrive_leader(uint64_t* bar, uint32_t rank) {
  if (rank == 0) mbar_arrive(bar);
  else mbar_arrive_cluster(bar, 0);
}

// ------------------------------------------------------------------------------------------- kernel
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1) k_fused3(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sG = base;                                    // [kSG][16 KB] generated A tiles
  uint8_t* sW = sG + kSG * kTile;                        // [kSW][16 KB] W1 / W2 half tiles
  uint8_t* sW3 = sW + kSW * kTile;                       // [kChunks][2 KB] W3 half (resident)
  uint8_t* sH2 = sW3 + kChunks * kW3Chunk;               // [4][16 KB] layer-3 A chunks
  Smem& S = *reinterpret_cast<Smem*>(sH2 + 4 * kTile);

  const uint32_t rank = cluster_ctarank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    const uint32_t two = rank == 0 ? 2u : 1u;
    for (int i = 0; i < kSG; i++) { mbar_init(&S.g_full[i], two); mbar_init(&S.g_empty[i], 1); }
    for (int i = 0; i < kSW; i++) { mbar_init(&S.w_full[i], two); mbar_init(&S.w_empty[i], 1); }
    mbar_init(&S.acc1_full, 1); mbar_init(&S.acc2_full, 1); mbar_init(&S.acc3_full, 1);
    mbar_init(&S.h1_ready, two); mbar_init(&S.acc2_free, two);
    for (int i = 0; i < 4; i++) { mbar_init(&S.h2c_full[i], two); mbar_init(&S.h2c_empty[i], 1); }
    S.base_g = -1;
    S.base_e = -1;
    fence_mbar_init();
  }
  if (warp == 1) { tmem_alloc2(&S.tbase, 512); tmem_relinquish2(); }
  // resident data: W3 half, biases (plain loads, once)
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.w3 + (size_t)rank * kChunks * kW3Chunk);
    uint4* dst = reinterpret_cast<uint4*>(sW3);
    for (int i = threadIdx.x; i < (int)(kChunks * kW3Chunk / 16); i += kThreads) dst[i] = src[i];
    for (int i = threadIdx.x; i < kN2; i += kThreads) S.b2[i] = a.b2[i];
    for (int i = threadIdx.x; i < kN3P; i += kThreads) S.b3[i] = i < a.n3 ? a.b3[i] : 0.f;
  }
  fence_proxy_async();
  fence_before();
  cluster_sync();
  fence_after();
  const uint32_t tb = S.tbase;
  const uint32_t R1 = tb, R2 = tb + 256u;

  if (warp == 0) {
    // ------------------------------------------------------------------ producer (both CTAs)
    if (lane == 0) {
      uint32_t ws = 0;
      const int nst = a.nkb1 + kNkb2;
      const uint8_t* src0 = a.wstream + (size_t)rank * nst * kTile;
      uint32_t tl = 0;
      for (uint64_t t = cluster; t < a.n_pairs_tiles; t += nclusters, tl++)
        for (int s = 0; s < nst; s++) {
          const uint32_t st = ws % kSW, ph = (ws / kSW) & 1u;
          mbar_wait(&S.w_empty[st], ph ^ 1u);
          if (s == 0) TR(tl, 31);
          mbar_expect_tx(&S.w_full[st], kTile);
          bulk_g2s(sW + st * kTile, src0 + (size_t)s * kTile, kTile, &S.w_full[st]);
          ws++;
        }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 1) {
      // ---------------------------------------------------------------- peer relay: W stages
      uint32_t ws = 0;
      const int nst = a.nkb1 + kNkb2;
      for (uint64_t t = cluster; t < a.n_pairs_tiles; t += nclusters)
        for (int s = 0; s < nst; s++) {
          const uint32_t st = ws % kSW, ph = (ws / kSW) & 1u;
          mbar_wait(&S.w_full[st], ph);
          mbar_arrive_cluster(&S.w_full[st], 0);
          ws++;
        }
    } else if (lane == 0 && rank == 0) {
      // ---------------------------------------------------------------- MMA issuer (leader)
      uint32_t gs = 0, ws = 0, tcount = 0;
      const uint32_t id1 = idesc_f16(256, kN1, 1, 1);     // bf16 x bf16 -> f32
      const uint32_t id2 = idesc_f16(256, kN2, 0, 0);     // f16 x f16 -> f32
      for (uint64_t t = cluster; t < a.n_pairs_tiles; t += nclusters, tcount++) {
        // layer 1 into R1 (in-order after the previous tile's layer 2 read R1)
        TR(tcount, 0);
        for (int kb = 0; kb < a.nkb1; kb++) {
          const uint32_t g = gs % kSG, w = ws % kSW;
          mbar_wait_cluster(&S.g_full[g], (gs / kSG) & 1u);
          if (kb < 13) TR(tcount, 16 + kb);
          mbar_wait_cluster(&S.w_full[w], (ws / kSW) & 1u);
          if (kb == 0) TR(tcount, 1);
          if (kb == a.nkb1 - 1) TR(tcount, 2);
          fence_after();
          const uint32_t ab = smem_u32(sG + g * kTile), bb = smem_u32(sW + w * kTile);
#pragma unroll
          for (int kk = 0; kk < 4; kk++)
            mma2_f16_ss(R1, sdesc_sw128(ab + 32u * kk), sdesc_sw128(bb + 32u * kk), id1, (kb | kk) ? 1u : 0u);
          mma2_commit(&S.g_empty[g], 0x3);
          mma2_commit(&S.w_empty[w], 0x3);
          gs++; ws++;
        }
        mma2_commit(&S.acc1_full, 0x3);
        // layer 2: A = H1 (fp16 hi | lo) in R1, B = W2 half tiles, D = R2
        mbar_wait_cluster(&S.h1_ready, tcount & 1u);
        TR(tcount, 3);
        mbar_wait_cluster(&S.acc2_free, (tcount & 1u) ^ 1u);
        TR(tcount, 4);
        fence_after();
        for (int kb = 0; kb < kNkb2; kb++) {
          const uint32_t w = ws % kSW;
          mbar_wait_cluster(&S.w_full[w], (ws / kSW) & 1u);
          fence_after();
          const uint32_t bb = smem_u32(sW + w * kTile);
#pragma unroll
          for (int kk = 0; kk < 4; kk++) {
            const uint32_t col = 32u * (2u * kb + (kk >> 1)) + 8u * (kk & 1);
            const uint64_t bd = sdesc_sw128(bb + 32u * kk);
            mma2_f16_ts(R2, R1 + col, bd, id2, (kb | kk) ? 1u : 0u);
            mma2_f16_ts(R2, R1 + col + 16u, bd, id2, 1u);
          }
          mma2_commit(&S.w_empty[w], 0x3);
          ws++;
        }
        mma2_commit(&S.acc2_full, 0x3);
        TR(tcount, 5);
      }
    }
  } else if (warp == 2) {
    if (lane == 0 && rank == 0) {
      // ---------------------------------------------------------------- layer-3 issuer (leader)
      uint32_t use[4] = {0, 0, 0, 0};
      const uint32_t id3 = idesc_f16(256, kN3P, 0, 0);
      uint32_t tl = 0;
      for (uint64_t t = cluster; t < a.n_pairs_tiles; t += nclusters, tl++) {
        for (int p = 0; p < kChunks; p++) {
          const int slot = 2 * (p & 1) + ((p >> 1) & 1);
          mbar_wait_cluster(&S.h2c_full[slot], use[slot] & 1u);
          if (p == 0) TR(tl, 14);
          use[slot]++;
          fence_after();
          const uint32_t ab = smem_u32(sH2 + slot * kTile), bb = smem_u32(sW3 + p * kW3Chunk);
#pragma unroll
          for (int kk = 0; kk < 4; kk++)
            mma2_f16_ss(R2, sdesc_sw128(ab + 32u * kk), sdesc_sw128(bb + 32u * kk), id3, (p | kk) ? 1u : 0u);
          mma2_commit(&S.h2c_empty[slot], 0x3);
        }
        mma2_commit(&S.acc3_full, 0x3);
        TR(tl, 15);
      }
    }
  } else if (warp >= 3 && warp < 7) {
    // ------------------------------------------------------------------ generator (both CTAs)
    const int r = threadIdx.x - 96;                        // row of this CTA's A tile
    uint32_t gs = 0;
    const uint32_t k0 = (uint32_t)a.pert.seed, k1 = (uint32_t)(a.pert.seed >> 32);
    const __nv_bfloat162 st2 = __floats2bfloat162_rn(a.pert.step_f, a.pert.step_f);
    const __nv_bfloat162 or2 = __floats2bfloat162_rn(a.pert.origin_f, a.pert.origin_f);
    const uint32_t step2 = *reinterpret_cast<const uint32_t*>(&st2), org2 = *reinterpret_cast<const uint32_t*>(&or2);
    const int n0 = a.n0;
    const int full_kb = n0 / 64;                           // K blocks made only of lattice pixels
    uint32_t tl = 0;
    for (uint64_t t = cluster; t < a.n_pairs_tiles; t += nclusters, tl++) {
      if (r == 0) TR(tl, 6);
      const TileInfo ti = tile_info(a, t);
      if (ti.b != S.base_g) {                              // stage the base image (bf16) once per base
        named_bar(1, 128);
        for (int i = r; i < (a.nkb1 * 64); i += 128) S.xg[i] = i < n0 ? a.bases[(size_t)ti.b * n0 + i] : (uint16_t)0;
        named_bar(1, 128);
        if (r == 0) S.base_g = ti.b;
      }
      const int grow = 128 * (int)rank + r;
      uint64_t c;
      if (a.eval_idx) c = grow < ti.nvalid ? a.eval_idx[ti.start + grow] : 0;
      else c = ti.start + (uint64_t)grow;
      const uint32_t c0 = (uint32_t)c, c1 = (uint32_t)(c >> 32), cb = (uint32_t)ti.b;
      for (int kb = 0; kb < a.nkb1; kb++) {
        const uint32_t st = gs % kSG, ph = (gs / kSG) & 1u;
        mbar_wait(&S.g_empty[st], ph ^ 1u);
        uint8_t* slot = sG + st * kTile;
        const uint4* xv = reinterpret_cast<const uint4*>(S.xg + 64 * kb);
        if (kb < full_kb) {
#pragma unroll
          for (int hb = 0; hb < 2; hb++) {
            const uint4 w = philox(c0, c1, cb, (uint32_t)(2 * kb + hb), k0, k1);
            const uint32_t wsr[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int ww = 0; ww < 4; ww++) {
              const int ch = 4 * hb + ww;                  // 16-byte chunk = 8 pixels
              *reinterpret_cast<uint4*>(slot + sw128_off(r, 16 * ch)) = lattice_word(wsr[ww], xv[ch], step2, org2);
            }
          }
        } else {
          // tail block: remaining pixels, then the bias columns (1.0) at K = n0 .. n0+2, then zeros
#pragma unroll
          for (int hb = 0; hb < 2; hb++) {
            const int j = 2 * kb + hb;
            uint4 w = make_uint4(0, 0, 0, 0);
            if (32 * j < n0) w = philox(c0, c1, cb, (uint32_t)j, k0, k1);
            const uint32_t wsr[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int ww = 0; ww < 4; ww++) {
              const int ch = 4 * hb + ww;
              const uint4 y = lattice_word(wsr[ww], xv[ch], step2, org2);
              uint32_t ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
              for (int k = 0; k < 4; k++) {
                const int e = 64 * kb + 8 * ch + 2 * k;     // K index of the low element
                uint32_t lo = ys[k] & 0xFFFFu, hi = ys[k] >> 16;
                if (e >= n0) lo = (e < n0 + 3) ? 0x3F80u : 0u;
                if (e + 1 >= n0) hi = (e + 1 < n0 + 3) ? 0x3F80u : 0u;
                ys[k] = lo | (hi << 16);
              }
              *reinterpret_cast<uint4*>(slot + sw128_off(r, 16 * ch)) = make_uint4(ys[0], ys[1], ys[2], ys[3]);
            }
          }
        }
        fence_proxy_async();
        named_bar(1, 128);
        if (r == 0) arrive_leader(&S.g_full[st], rank);
        gs++;
      }
      if (r == 0) TR(tl, 7);
    }
  } else if (warp >= 7) {
    // ------------------------------------------------------------------ epilogue (both CTAs)
    const int e = threadIdx.x - 224;                       // 0..255
    const int grp = e >> 7;                                // 0 or 1
    const int quad = warp & 3;
    const int r = 32 * quad + lane;                        // row = TMEM lane
    const uint32_t loff = (uint32_t)(32 * quad) << 16;
    uint32_t tcount = 0, h2use[2] = {0, 0};
    const float tg2 = a.cov.tg_f[1], tg3 = a.cov.tg_f[2], th1 = a.cov.th_f[0], th2 = a.cov.th_f[1];
    float tau[3];
#pragma unroll
    for (int l = 0; l < 3; l++) tau[l] = a.cov.tau_dev ? a.cov.tau_dev[l] : a.cov.tau[l];
    const bool eval = a.eval_idx != nullptr;
    for (uint64_t t = cluster; t < a.n_pairs_tiles; t += nclusters, tcount++) {
      const TileInfo ti = tile_info(a, t);
      const int grow = 128 * (int)rank + r;
      const bool valid = grow < ti.nvalid;
      const uint64_t cidx = a.eval_idx ? (valid ? (uint64_t)(ti.start + grow) : 0) : ti.start + (uint64_t)grow;
      if (ti.b != S.base_e) {                              // stage the base trace once per base
        named_bar(2, 256);
        const float* tr = a.trace + (size_t)ti.b * a.T;
        for (int i = e; i < kN1; i += 256) S.ub1[i] = tr[i];
        for (int i = e; i < kN2; i += 256) S.ub2[i] = tr[kN1 + i];
        for (int i = e; i < kN3P; i += 256) S.ub3[i] = i < a.n3 ? tr[kN1 + kN2 + i] : 0.f;
        named_bar(2, 256);
        if (e < 17) {
          const float* u = e < 8 ? S.ub1 + 32 * e : (e < 16 ? S.ub2 + 32 * (e - 8) : S.ub3);
          uint32_t m = 0;
          for (int i = 0; i < 32; i++) m |= (__float_as_uint(u[i]) >> 31) << i;
          if (e < 8) S.nb1[e] = m; else if (e < 16) S.nb2[e - 8] = m; else S.nb3 = m & ((a.n3 >= 32) ? ~0u : ((1u << a.n3) - 1u));
        } else if (e < 20) {
          const int l = e - 17;
          const int n = l == 0 ? kN1 : (l == 1 ? kN2 : a.n3);
          const float* u = l == 0 ? S.ub1 : (l == 1 ? S.ub2 : S.ub3);
          float m = 3.0e38f;
          for (int i = 0; i < n; i++) m = fminf(m, fabsf(u[i]));
          S.minub[l] = m;
        }
        named_bar(2, 256);
        if (e == 0) S.base_e = ti.b;
      }
      // =========================== E1: layer-1 potentials -> predicates, H1 (fp16 hi|lo) in place
      mbar_wait(&S.acc1_full, tcount & 1u);
      if (e == 0) TR(tcount, 8);
      fence_after();
      int nsc = 0, first = -1;
      uint32_t fw = 0;
      float linf = 0.f, minab = 3.0e38f;
#pragma unroll 1
      for (int pi = 0; pi < 4; pi++) {
        const int p = 4 * grp + pi;
        uint32_t v[32];
        tmem_ld32(R1 + loff + 32u * p, v);
        tmem_ld_wait();
        uint32_t neg = 0;
#pragma unroll
        for (int i = 0; i < 32; i++) neg |= (v[i] >> 31) << i;
        const uint32_t scw = neg ^ S.nb1[p];
        nsc += __popc(scw);
        if (first < 0 && scw) { first = p; fw = scw; }
        const float4* ub = reinterpret_cast<const float4*>(S.ub1 + 32 * p);
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const float4 b4 = ub[q];
          const float u0 = __uint_as_float(v[4 * q]), u1 = __uint_as_float(v[4 * q + 1]);
          const float u2 = __uint_as_float(v[4 * q + 2]), u3 = __uint_as_float(v[4 * q + 3]);
          linf = fmaxf(linf, fmaxf(fmaxf(fabsf(u0 - b4.x), fabsf(u1 - b4.y)), fmaxf(fabsf(u2 - b4.z), fabsf(u3 - b4.w))));
          minab = fminf(minab, fminf(fminf(fabsf(u0), fabsf(u1)), fminf(fabsf(u2), fabsf(u3))));
        }
        if (eval && valid) {
#pragma unroll
          for (int i = 0; i < 32; i++) a.eval_out[cidx * a.T + 32 * p + i] = __uint_as_float(v[i]);
        }
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int k = 0; k < 16; k++) split_pair(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]), hi[k], lo[k]);
        tmem_st16(R1 + loff + 32u * p, hi);
        tmem_st16(R1 + loff + 32u * p + 16u, lo);
      }
      tmem_st_wait();
      S.x_nsc[grp][r] = nsc; S.x_first[grp][r] = first; S.x_fw[grp][r] = fw;
      S.x_linf[grp][r] = linf; S.x_minab[grp][r] = minab;
      fence_before();
      if (e == 0) TR(tcount, 9);
      if (e == 128) TR(tcount, 29);
      named_bar(2, 256);
      if (e == 0) arrive_leader(&S.h1_ready, rank);
      // combine the two groups' summaries of layer 1
      const int o = grp ^ 1;
      const int nsc1 = nsc + S.x_nsc[o][r];
      int f1;
      uint32_t fw1;
      if (grp == 0) { f1 = first >= 0 ? first : S.x_first[1][r]; fw1 = first >= 0 ? fw : S.x_fw[1][r]; }
      else { f1 = S.x_first[0][r] >= 0 ? S.x_first[0][r] : first; fw1 = S.x_first[0][r] >= 0 ? S.x_fw[0][r] : fw; }
      const int istar1 = f1 >= 0 ? 32 * f1 + __ffs(fw1) - 1 : -1;
      const float linf1 = fmaxf(linf, S.x_linf[o][r]);
      const float minab1 = fminf(fminf(minab, S.x_minab[o][r]), S.minub[0]);
      const bool cond1 = (nsc1 == 1) || (nsc1 == 0 && linf1 >= th1);
      const bool amb1 = minab1 < tau[0] || (nsc1 == 0 && fabsf(linf1 - th1) < tau[0]);
      // =========================== E2: layer-2 potentials -> predicates, H2 chunks for layer 3
      mbar_wait(&S.acc2_full, tcount & 1u);
      if (e == 0) TR(tcount, 10);
      fence_after();
      const bool pair12 = a.pair12 >= 0 && cond1 && valid && !eval;
      const bool any12 = __any_sync(0xffffffffu, pair12);
      int nsc2 = 0, first2 = -1;
      uint32_t fw2 = 0;
      float linf2 = 0.f, minab2 = 3.0e38f, vcamb2 = 3.0e38f;
      uint32_t scs[4], vcs[4];
#pragma unroll 1
      for (int pi = 0; pi < 4; pi++) {
        const int p = 2 * pi + grp;                        // group g takes pieces of parity g
        uint32_t v[32];
        tmem_ld32(R2 + loff + 32u * p, v);
        tmem_ld_wait();
        float u[32];
        const float4* bb = reinterpret_cast<const float4*>(S.b2 + 32 * p);
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const float4 b4 = bb[q];
          u[4 * q] = __uint_as_float(v[4 * q]) + b4.x;
          u[4 * q + 1] = __uint_as_float(v[4 * q + 1]) + b4.y;
          u[4 * q + 2] = __uint_as_float(v[4 * q + 2]) + b4.z;
          u[4 * q + 3] = __uint_as_float(v[4 * q + 3]) + b4.w;
        }
        uint32_t neg = 0;
#pragma unroll
        for (int i = 0; i < 32; i++) neg |= (__float_as_uint(u[i]) >> 31) << i;
        const uint32_t scw = neg ^ S.nb2[p];
        nsc2 += __popc(scw);
        if (first2 < 0 && scw) { first2 = p; fw2 = scw; }
        const float4* ub = reinterpret_cast<const float4*>(S.ub2 + 32 * p);
        uint32_t vcw = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const float4 b4 = ub[q];
          const float d0 = fabsf(u[4 * q] - b4.x), d1 = fabsf(u[4 * q + 1] - b4.y);
          const float d2 = fabsf(u[4 * q + 2] - b4.z), d3 = fabsf(u[4 * q + 3] - b4.w);
          linf2 = fmaxf(linf2, fmaxf(fmaxf(d0, d1), fmaxf(d2, d3)));
          minab2 = fminf(minab2, fminf(fminf(fabsf(u[4 * q]), fabsf(u[4 * q + 1])), fminf(fabsf(u[4 * q + 2]), fabsf(u[4 * q + 3]))));
          if (any12) {
            const float dd[4] = {d0, d1, d2, d3};
#pragma unroll
            for (int k = 0; k < 4; k++) {
              if (dd[k] >= tg2) vcw |= 1u << (4 * q + k);
              vcamb2 = fminf(vcamb2, fabsf(dd[k] - tg2));
            }
          }
        }
        scs[pi] = scw;
        vcs[pi] = vcw & ~scw;
        if (eval && valid) {
#pragma unroll
          for (int i = 0; i < 32; i++) a.eval_out[cidx * a.T + kN1 + 32 * p + i] = u[i];
        }
        // stage [hi 32 | lo 32] of this piece as layer-3 A chunk p
        const int slot = 2 * grp + (pi & 1);
        mbar_wait(&S.h2c_empty[slot], (h2use[pi & 1] & 1u) ^ 1u);
        h2use[pi & 1]++;
        uint8_t* dst = sH2 + slot * kTile;
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int k = 0; k < 16; k++) split_pair(u[2 * k], u[2 * k + 1], hi[k], lo[k]);
#pragma unroll
        for (int m = 0; m < 4; m++) {
          *reinterpret_cast<uint4*>(dst + sw128_off(r, 16 * m)) = make_uint4(hi[4 * m], hi[4 * m + 1], hi[4 * m + 2], hi[4 * m + 3]);
          *reinterpret_cast<uint4*>(dst + sw128_off(r, 64 + 16 * m)) = make_uint4(lo[4 * m], lo[4 * m + 1], lo[4 * m + 2], lo[4 * m + 3]);
        }
        fence_proxy_async();
        fence_before();
        named_bar(3 + grp, 128);
        if ((e & 127) == 0) arrive_leader(&S.h2c_full[slot], rank);
      }
      // combine summaries of layer 2 and finish pair (1, 2)
      S.x_nsc[grp][r] = nsc2; S.x_first[grp][r] = first2; S.x_fw[grp][r] = fw2;
      S.x_linf[grp][r] = linf2; S.x_minab[grp][r] = minab2; S.x_vcamb[grp][r] = vcamb2;
      if (e == 128) TR(tcount, 30);
      named_bar(2, 256);
      if (e == 0) TR(tcount, 11);
      const int nsc2t = nsc2 + S.x_nsc[o][r];
      int f2 = first2;
      uint32_t fw2t = fw2;
      if (S.x_first[o][r] >= 0 && (f2 < 0 || S.x_first[o][r] < f2)) { f2 = S.x_first[o][r]; fw2t = S.x_fw[o][r]; }
      const int istar2 = f2 >= 0 ? 32 * f2 + __ffs(fw2t) - 1 : -1;
      const float linf2t = fmaxf(linf2, S.x_linf[o][r]);
      const float minab2t = fminf(fminf(minab2, S.x_minab[o][r]), S.minub[1]);
      const float vcamb2t = fminf(vcamb2, S.x_vcamb[o][r]);
      if (pair12) {
        const bool certain = !amb1 && minab2t >= tau[1] && vcamb2t >= tau[1];
        const uint32_t* off = a.cov.off[a.pair12];
#pragma unroll
        for (int pi = 0; pi < 4; pi++) {
          const int p = 2 * pi + grp;
          const uint32_t sw = scs[pi], vw = vcs[pi];
          uint32_t is, iv;
          if (nsc1 == 1) { is = off[0] + istar1 * 8 + p; iv = off[1] + istar1 * 8 + p; }
          else { is = off[2] + p; iv = off[3] + p; }
          if (sw) { atomicOr(&a.res.cov_all[is], sw); if (certain) atomicOr(&a.res.cov_certain[is], sw); }
          if (vw) { atomicOr(&a.res.cov_all[iv], vw); if (certain) atomicOr(&a.res.cov_certain[iv], vw); }
        }
      }
      const bool cond2 = (nsc2t == 1) || (nsc2t == 0 && linf2t >= th2);
      const bool amb2 = minab2t < tau[1] || (nsc2t == 0 && fabsf(linf2t - th2) < tau[1]);
      // =========================== E3: logits -> pair (2, 3), argmax, property, counts (group 0)
      if (grp == 0) {
        mbar_wait(&S.acc3_full, tcount & 1u);
        if (e == 0) TR(tcount, 12);
        fence_after();
        uint32_t v[16];
        tmem_ld16(R2 + loff, v);
        tmem_ld_wait();
        fence_before();
        named_bar(3, 128);
        if (e == 0) arrive_leader(&S.acc2_free, rank);
        const int n3 = a.n3;
        float y[16];
#pragma unroll
        for (int i = 0; i < 16; i++) y[i] = __uint_as_float(v[i]) + S.b3[i];
        if (eval) {
          if (valid)
            for (int i = 0; i < n3; i++) a.eval_out[cidx * a.T + kN1 + kN2 + i] = y[i];
        } else {
          const int bcls = a.cls[ti.b];
          // pair (2, 3)
          if (a.pair23 >= 0 && cond2 && valid) {
            uint32_t neg = 0, vcw = 0;
            float minab3 = S.minub[2], vcamb3 = 3.0e38f;
#pragma unroll
            for (int i = 0; i < 16; i++)
              if (i < n3) {
                neg |= (__float_as_uint(y[i]) >> 31) << i;
                const float d = fabsf(y[i] - S.ub3[i]);
                if (d >= tg3) vcw |= 1u << i;
                vcamb3 = fminf(vcamb3, fabsf(d - tg3));
                minab3 = fminf(minab3, fabsf(y[i]));
              }
            const uint32_t scw = neg ^ S.nb3;
            const uint32_t vw = vcw & ~scw;
            const bool certain = !amb2 && minab3 >= tau[2] && vcamb3 >= tau[2];
            const uint32_t* off = a.cov.off[a.pair23];
            uint32_t is, iv;
            if (nsc2t == 1) { is = off[0] + istar2; iv = off[1] + istar2; }
            else { is = off[2]; iv = off[3]; }
            if (scw) { atomicOr(&a.res.cov_all[is], scw); if (certain) atomicOr(&a.res.cov_certain[is], scw); }
            if (vw) { atomicOr(&a.res.cov_all[iv], vw); if (certain) atomicOr(&a.res.cov_certain[iv], vw); }
          }
          // argmax (lowest index on ties), margin, property
          int cls = 0;
          float top1 = y[0];
#pragma unroll
          for (int i = 1; i < 16; i++) if (i < n3 && y[i] > top1) { top1 = y[i]; cls = i; }
          bool viol = false, flag = false;
          if (a.prop.kind == MLPV_PROP_THRESHOLD_LITERAL) {
            const int D = a.prop.target >= 0 ? a.prop.target : bcls;
            bool any = false;
            float yD = 0.f;
#pragma unroll
            for (int i = 0; i < 16; i++)
              if (i < n3) {
                if (i == D) yD = y[i];
                if (i != D && y[i] > a.prop.V_f) any = true;
                if (fabsf(y[i] - a.prop.V_f) < a.cov.near_tie) flag = true;
              }
            viol = yD < a.prop.V_f && any;
          } else {
            float top2 = -3.0e38f;
#pragma unroll
            for (int i = 0; i < 16; i++) if (i < n3 && i != cls && y[i] > top2) top2 = y[i];
            flag = n3 > 1 && top1 - top2 < a.cov.near_tie;
            viol = a.prop.kind == MLPV_PROP_TARGET_NEVER ? cls == a.prop.target : cls != bcls;
          }
          if (!valid) { viol = false; flag = false; }
          const uint32_t nv = __reduce_add_sync(0xffffffffu, viol ? 1u : 0u);
          const uint32_t nf = __reduce_add_sync(0xffffffffu, flag ? 1u : 0u);
          const uint32_t nc = __reduce_add_sync(0xffffffffu, valid ? 1u : 0u);
          const uint32_t rel = viol ? (uint32_t)grow : 0xFFFFFFFFu;
          const uint32_t relu = (viol && !flag) ? (uint32_t)grow : 0xFFFFFFFFu;
          const uint32_t mn = __reduce_min_sync(0xffffffffu, rel), mnu = __reduce_min_sync(0xffffffffu, relu);
          if (lane == 0) {
            if (nc) atomicAdd(reinterpret_cast<unsigned long long*>(a.res.checked) + ti.b, (unsigned long long)nc);
            if (nv) atomicAdd(reinterpret_cast<unsigned long long*>(a.res.violated) + ti.b, (unsigned long long)nv);
            if (nf) atomicAdd(reinterpret_cast<unsigned long long*>(a.res.flagged) + ti.b, (unsigned long long)nf);
            if (mn != 0xFFFFFFFFu) atomicMin(reinterpret_cast<unsigned long long*>(a.res.first_cex) + ti.b, (unsigned long long)(ti.start + mn));
            if (mnu != 0xFFFFFFFFu) atomicMin(reinterpret_cast<unsigned long long*>(a.res.first_cex_unflagged) + ti.b, (unsigned long long)(ti.start + mnu));
          }
        }
        if (e == 0) TR(tcount, 13);
      }
    }
  }
  fence_before();
  __syncthreads();
  cluster_sync();
  fence_after();
  if (warp == 1) tmem_dealloc2(tb, 512);
}

}  // namespace f3

#ifdef MLPV_TRACE
extern "C" int mlpv_f3_trace_read(void* host) {
  return (int)cudaMemcpyFromSymbol(host, f3::g_trace, sizeof f3::g_trace);
}
#endif

// ------------------------------------------------------------------------------------------- host
bool fused3_applicable(const DevNet& net) {
  return net.numeric == MLPV_NUM_BF16 && net.L == 3 && net.sizes[1] == f3::kN1 && net.sizes[2] == f3::kN2 &&
         net.sizes[3] <= 16 && net.sizes[0] % 2 == 0 && net.sizes[0] + 3 <= f3::kMaxN0;
}

static size_t sw128_h(uint32_t row, uint32_t byte) {
  return (row >> 3) * 1024u + (row & 7u) * 128u + ((((byte >> 4) ^ row) & 7u) << 4) + (byte & 15u);
}
static uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}
static float bf2f(uint16_t b) {
  const uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static uint16_t f2h(float f) {
  const __half h = __float2half_rn(f);
  uint16_t u;
  memcpy(&u, &h, 2);
  return u;
}

// Weight layouts of k_fused3 (host-side, once per handle):
//   stream [rank][nkb1 + 4][16 KB]: W1 rows [128 rank, +128) per K block (bias hi/mid/lo at K = n0..n0+2),
//          then W2 (fp16) rows [128 rank, +128) per K block of 64 layer-1 neurons;
//   w3 [rank][8][2 KB]: W3 (fp16) rows [16 rank, +16) (rows >= n3 zero), chunk p = [W3[:, 32p..] | same].
cudaError_t prepare_fused3(const DevNet& net, const void* const* W_host, const void* const* b_host, void** stream_dev,
                           void** w3_dev) {
  const int n0 = net.sizes[0], n3 = net.sizes[3];
  const int nkb1 = (2 * (n0 + 3) + 127) / 128;
  const int nst = nkb1 + f3::kNkb2;
  std::vector<uint8_t> st((size_t)2 * nst * f3::kTile, 0), w3((size_t)2 * f3::kChunks * f3::kW3Chunk, 0);
  const uint16_t* W1 = static_cast<const uint16_t*>(W_host[0]);
  const uint16_t* W2 = static_cast<const uint16_t*>(W_host[1]);
  const uint16_t* W3 = static_cast<const uint16_t*>(W_host[2]);
  const float* b1 = static_cast<const float*>(b_host[0]);
  auto put16 = [&](uint8_t* tile, int row, int kelem, uint16_t v) {
    const size_t o = sw128_h((uint32_t)row, (uint32_t)(2 * (kelem % 64)));
    tile[o] = (uint8_t)(v & 0xFF);
    tile[o + 1] = (uint8_t)(v >> 8);
  };
  for (int rk = 0; rk < 2; rk++) {
    for (int rr = 0; rr < 128; rr++) {
      const int n = 128 * rk + rr;
      for (int k = 0; k < n0 + 3; k++) {
        uint16_t v;
        if (k < n0) v = W1[(size_t)n * n0 + k];
        else {
          const float b = b1[n];
          const uint16_t p1 = f2bf(b);
          const float r1 = b - bf2f(p1);
          const uint16_t p2 = f2bf(r1);
          const float r2 = r1 - bf2f(p2);
          v = k == n0 ? p1 : (k == n0 + 1 ? p2 : f2bf(r2));
        }
        put16(st.data() + ((size_t)rk * nst + k / 64) * f3::kTile, rr, k, v);
      }
      for (int k = 0; k < f3::kN1; k++) {
        const uint16_t h = f2h(bf2f(W2[(size_t)n * f3::kN1 + k]));      // exact for |w| >= 2^-17
        put16(st.data() + ((size_t)rk * nst + nkb1 + k / 64) * f3::kTile, rr, k, h);
      }
    }
    for (int rr = 0; rr < 16; rr++) {
      const int n = 16 * rk + rr;
      for (int p = 0; p < f3::kChunks; p++)
        for (int i = 0; i < 32; i++) {
          const uint16_t h = n < n3 ? f2h(bf2f(W3[(size_t)n * f3::kN2 + 32 * p + i])) : (uint16_t)0;
          uint8_t* tile = w3.data() + ((size_t)rk * f3::kChunks + p) * f3::kW3Chunk;
          for (int half = 0; half < 2; half++) {
            const size_t o = sw128_h((uint32_t)rr, (uint32_t)(64 * half + 2 * i));
            tile[o] = (uint8_t)(h & 0xFF);
            tile[o + 1] = (uint8_t)(h >> 8);
          }
        }
    }
  }
  cudaError_t e = cudaMalloc(stream_dev, st.size());
  if (e != cudaSuccess) return e;
  e = cudaMemcpy(*stream_dev, st.data(), st.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return e;
  e = cudaMalloc(w3_dev, w3.size());
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*w3_dev, w3.data(), w3.size(), cudaMemcpyHostToDevice);
}

cudaError_t launch_fused3(const DevNet& net, const void* stream_w, const void* w3, const void* bases, int n_base,
                          const DevPert& pert, const DevProp& prop, const DevCov& cov, const DevResult& res,
                          BaseWS ws, const uint64_t* eval_idx, int64_t eval_n, int eval_base, void* eval_out,
                          int num_sms, cudaStream_t st) {
  f3::Args a;
  memset(&a, 0, sizeof a);
  a.n0 = net.sizes[0];
  a.n3 = net.sizes[3];
  a.nkb1 = (2 * (a.n0 + 3) + 127) / 128;
  a.wstream = static_cast<const uint8_t*>(stream_w);
  a.w3 = static_cast<const uint8_t*>(w3);
  a.b2 = static_cast<const float*>(net.b[1]);
  a.b3 = static_cast<const float*>(net.b[2]);
  a.bases = static_cast<const uint16_t*>(bases);
  a.pert = pert; a.prop = prop; a.cov = cov; a.res = res;
  a.trace = static_cast<const float*>(ws.trace);
  a.cls = ws.cls;
  a.T = net.trace_len;
  a.pair12 = a.pair23 = -1;
  for (int p = 0; p < cov.n_pairs; p++) {
    if (cov.lower[p] == 1) a.pair12 = p;
    if (cov.lower[p] == 2) a.pair23 = p;
  }
  a.eval_idx = eval_idx; a.eval_n = eval_n; a.eval_base = eval_base; a.eval_out = static_cast<float*>(eval_out);
  if (eval_idx) {
    a.tiles_per_base = (uint64_t)((eval_n + 255) / 256);
    a.n_pairs_tiles = a.tiles_per_base;
  } else {
    a.tiles_per_base = (pert.end - pert.begin + 255) / 256;
    a.n_pairs_tiles = a.tiles_per_base * (uint64_t)n_base;
  }
  if (a.n_pairs_tiles == 0) return cudaSuccess;
  uint64_t nclusters = (uint64_t)(num_sms / 2);
  if (nclusters > a.n_pairs_tiles) nclusters = a.n_pairs_tiles;
  cudaError_t e = cudaFuncSetAttribute(f3::k_fused3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f3::kSmemBytes);
  if (e != cudaSuccess) return e;
  f3::k_fused3<<<(unsigned)(2 * nclusters), f3::kThreads, f3::kSmemBytes, st>>>(a);
  return cudaGetLastError();
}

}  // namespace mlpv
