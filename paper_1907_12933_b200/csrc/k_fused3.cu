// k_fused3.cu -- the specialised large-net kernel for 3-layer bf16 nets with 256-wide hidden layers
// (BASELINE config 4: 784-256-256-10), SURVEY.md §8(a) rows a1-a9 in one persistent launch.
//
// A CTA pair (cluster of 2) owns a contiguous range of 256-candidate pair tiles; the leader
// (cluster rank 0) issues every tcgen05.mma with cta_group::2 (M = 256: rows 0-127 of the tile in
// CTA 0's TMEM lanes, rows 128-255 in CTA 1's), each CTA supplying half of every B operand.
//
//   layer 1  the exact L-inf box lattice (PHILOX_BOX, reading C14b) is linear in the Philox levels,
//            u1 = W1 x + b1 + origin W1 1 + step W1 l: A = the levels l of every pixel (fp16
//            subnormals l * 2^-24, one PRMT per pixel pair) generated on chip into a SWIZZLE_128B
//            ring; B = W1 (fp16) half tiles streamed by cp.async.bulk; TMEM cols [0,256) accumulate
//            2^-24 W1 l and E1 forms u1 = base1 + (step 2^24) acc with base1 from the prologue.
//   E1       8 warps (two per TMEM lane quadrant, "halves"), thread = candidate row; one pass, one
//            32-neuron piece per step: u1, h1 = ReLU(u1) -> fp16 [hi | lo] in place (reading C19),
//            the sign-change bits against the base potentials, and the L-inf / min|u| partials
//            while some row of the warp can still end with <= 1 change (the only case a covering
//            method fires on).  Half 0 takes pieces 0,1,2,4,6 and starts at once; half 1 first
//            finishes the previous tile's E3, then takes 3,5,7.  Each piece signs off its part of
//            a 64-neuron K block of layer 2.
//   layer 2  A = H1 straight from TMEM, B = W2 (fp16, the same tile for hi and lo); the bias is one
//            more SS MMA (ones column x [b_hi | b_lo]); accumulator TMEM cols [256,512).
//   E2       pass A: sign words sc2 and counts; pass B: u2 -> [hi | lo] in place, one piece per step
//            (neurons 240-255 go to a small shared-memory tile so that their 16 columns can hold
//            the layer-3 accumulator).  The layer-2 statistics are needed by < 1 % of the rows: a
//            warp's (up to 4) such rows are evaluated by all 32 lanes, one row at a time, from
//            shared-memory copies; warps with more compute them per lane.  Then the pair-(1,2)
//            coverage words.
//   layer 3  N = 16 (n_3 <= 16): A = H2 from TMEM (and the tail tile), accumulator TMEM cols
//            [496,512); issued by the MMA issuer between layer-1 stages of the next tile.
//   E3       half 1: logits, pair (2,3), argmax / margin / property, counts, first counterexample.
//
// Warp roles (24 warps, see kW* below): 0-11 generator (three warpgroups taking ring stages in
// turn), 12-19 epilogue team, 20 idle, 21 weight producer, 23 MMA issuer of all layers (leader) /
// weight relay (peer) and TMEM owner.  DESIGN.md §6 has the measured timeline.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <type_traits>
#include <cstring>
#include <string>
#include <vector>

#include "mlpv_internal.cuh"
#include "tc_ptx.cuh"

namespace mlpv {
using namespace tc;

namespace f3 {
#ifndef MLPV_EXP
#define MLPV_EXP 0                           // timing experiments only (tools/exp_f3.sh); 0 = product
#endif
// MLPV_EXP = 21: the generators skip their shared-memory stores; 104: the weights are streamed
// only for the first tile (results are wrong in both; they isolate a resource in the timeline)
#ifdef MLPV_TRACE
// debug timeline (tools/trace_fused3.py): clock64 stamps of the first 64 tiles of cluster 0
__device__ unsigned long long g_trace[2][64][32];
#define TR(tl, ev) do { if (cluster == 0 && (tl) < 64) g_trace[rank][(tl)][(ev)] = clock64(); } while (0)
// issuer detail: [tile 8..11][kb 0..12][0 top, 1 after throttle, 2 after g_full, 3 after w_full]
__device__ unsigned long long g_trace_iss[4][13][8];
// epilogue detail: [0 E1 / 1 E2][tile 8..11][0 start, 1 pass A done, 2..5 kb signals, 6 end]
__device__ unsigned long long g_trace_epi[2][4][8];
#define TRE(team, tl, ev) do { if (cluster == 0 && rank == 0 && et == 0 && (tl) >= 8 && (tl) < 12) \
    g_trace_epi[(team)][(tl) - 8][(ev)] = clock64(); } while (0)
// per-warp epilogue detail for tile 9: [rank][epilogue warp][0 E1 / 1 E2][0 start, 1 signs exchanged,
// 2..5 K-block signals (E1: own pieces in order; E2: the blocks this half signals), 6 end]
__device__ unsigned long long g_trace_e2[2][8][2][8];
#define TRE2(tl, team, ev) do { if (cluster == 0 && lane == 0 && (tl) == 9) \
    g_trace_e2[rank][warp - kWE][(team)][(ev)] = clock64(); } while (0)
// E2 pass B per group, tile 9, rank 0, all 8 epilogue warps: [warp][i][0 top, 1 after stats, 2 after split, 3 after stores/signal, 4 after ld wait]
__device__ unsigned long long g_trace_grp[8][8][5];
#define TRP(tl, i, ev) do { if (cluster == 0 && rank == 0 && lane == 0 && (tl) == 9) \
    g_trace_grp[warp - kWE][(i)][(ev)] = clock64(); } while (0)
// E1 per piece, tile 9, cluster 0: [rank][epilogue warp][piece step][0 top, 1 ld done, 2 computed, 3 signed off]
__device__ unsigned long long g_trace_e1p[2][8][5][4];
#define TR1(tl, i, ev) do { if (cluster == 0 && lane == 0 && (tl) == 9) \
    g_trace_e1p[rank][warp - kWE][(i)][(ev)] = clock64(); } while (0)
// completion time of every layer-1 stage of tiles 8..11 (observed by the idle warp 3)
__device__ unsigned long long g_trace_done[4][13];
#define TRI(tl, kb, ev) do { if (cluster == 0 && (tl) >= 8 && (tl) < 12) g_trace_iss[(tl) - 8][(kb)][(ev)] = clock64(); } while (0)
// generator detail: [rank][h][tile 8..11][kb 0..12][event 0..4]
__device__ unsigned long long g_trace_gen[2][2][4][13][5];
#define TRG(tl, kb, ev) do { if (cluster == 0 && lane == 0 && (gw & 3) == 0 && (tl) >= 8 && (tl) < 12) \
    g_trace_gen[rank][grp][(tl) - 8][(kb)][(ev)] = clock64(); } while (0)
#else
#define TR(tl, ev) do { } while (0)
#define TRG(tl, kb, ev) do { } while (0)
#define TRI(tl, kb, ev) do { } while (0)
#define TRE(team, tl, ev) do { } while (0)
#define TRE2(tl, i, ev) do { } while (0)
#define TRP(tl, i, ev) do { } while (0)
#define TR1(tl, i, ev) do { } while (0)
#endif

constexpr int kThreads = 768;
// ring depths and E2's after-hand-off statistics rows are compile-time parameters (measured, cfg4,
// 3 interleaved A/B runs each: 5 generator stages + up to 4 statistics rows per warp +1.5 % over the
// round-2 6 stages + 1 row; 5 stages alone -0.5 %, 6 + 4 with a 4-stage W ring and 5 + 5: no better)
#ifndef MLPV_F3_SG
#define MLPV_F3_SG 5
#endif
#ifndef MLPV_F3_C1ROWS
#define MLPV_F3_C1ROWS 4
#endif
constexpr int kSG = MLPV_F3_SG;              // generator ring stages
constexpr int kC1Rows = MLPV_F3_C1ROWS;      // E2: statistics rows per warp evaluated after the hand-off
#ifndef MLPV_F3_SW
#define MLPV_F3_SW 5
#endif
constexpr int kSW = MLPV_F3_SW;              // weight ring stages
constexpr uint32_t kBiasTile = 4096;         // 128 rows x K 16 (fp16), no-swizzle layout
constexpr uint32_t kTile = 16384;            // 128 rows x 128 B
constexpr int kN1 = 256, kN2 = 256, kN3P = 16;
constexpr int kNkb2 = kN1 / 64;              // W2 K blocks (64 fp16 per 128-B row)
constexpr int kChunks = kN2 / 32;            // layer-3 chunks (32 neurons of layer 2)
constexpr uint32_t kW3Chunk = 8u * 128u;     // per CTA: 8 rows x 128 B
constexpr int kMaxN0 = 1024;
// Warp roles (six warpgroups; setmaxnreg moves registers from the generator and control groups to
// the epilogues).  The SMSP arbiter issues the highest warp id first (B300_MICROARCH.md,
// "Multi-warp arbiter"), so the roles are stacked by how latency-critical they are: 20-23 control
// (20 idle / trace observer, 21 weight producer, 23 MMA issuer for all three layers / TMEM owner),
// 12-19 epilogue team (E1, E2, E3 -- on the tile's critical path; two warps per TMEM lane quadrant),
// 0-11 generator (throughput work with a five-stage ring of slack; one warpgroup per stage group).
#ifndef MLPV_F3_GEN_SLEEP
#define MLPV_F3_GEN_SLEEP 128
#endif
#if MLPV_EXP == 31
constexpr int kNGenGroups = 2, kWE = 12, kWIdle = 20, kWProd = 21, kWIss = 23;   // timing experiment: warps 8-11 idle
#else
constexpr int kNGenGroups = 3, kWE = 12, kWIdle = 20, kWProd = 21, kWIss = 23;   // warp 22: spare
#endif
// (Measured and kept: three generator groups.  Two groups keep up as well (MLPV_EXP 31, same tile
// period); a 2-generator / 3-epilogue-warpgroup variant with 3-way row exchanges (E1 on three
// warps per quadrant) ran 0.7 % slower: E1's pieces took proportionally longer per warp -- the step
// is bound by the SMSPs' shared issue / TMEM traffic, not by the warp count.)
__host__ __device__ constexpr int gen_index(int warp) { return warp; }
// setmaxnreg only redistributes the CTA's launch allocation (768 threads x kRegLaunch, checked at
// launch): 3 generator + 2 epilogue + 1 control warpgroups must fit in 6 x kRegLaunch per thread.
constexpr int kRegLaunch = 80, kRegGen = 72, kRegEpi = 96;
static_assert(4 * kRegGen + 2 * kRegEpi <= 6 * kRegLaunch, "setmaxnreg budget");

// device weight block of one handle: [rank][nst][16 KB] stream | [rank][8][1 KB] W3 | ones | [rank] bias2
struct Layout {
  size_t stream, w3, ones, bias2, total;
  int nkb1, nk16, nst;
};
__host__ __device__ inline Layout layout_of(int n0) {
  Layout L;
  L.nk16 = (n0 + 15) / 16;                   // K steps of layer 1 (the bias enters through base1)
  L.nkb1 = (L.nk16 + 3) / 4;
  L.nst = L.nkb1 + kNkb2;
  L.stream = 0;
  L.w3 = L.stream + (size_t)2 * L.nst * kTile;
  L.ones = L.w3 + (size_t)2 * kChunks * kW3Chunk;
  L.bias2 = L.ones + kBiasTile;
  L.total = L.bias2 + 2 * (size_t)kBiasTile;
  return L;
}

struct Args {
  int n0, n3, nkb1, nk16;
  uint64_t n_pairs_tiles, tiles_per_base;
  const uint8_t* wblk;                       // Layout above
  Layout lay;
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
  float stepS;                               // u1 = base1 + stepS * acc: PHILOX_BOX step * 2^24, PHILOX_CLAMP 2^-s
  const float* base1;                        // [n_base][256] W1 x + b1 (+ origin W1 1 for PHILOX_BOX)
  int clamp;                                 // PHILOX_CLAMP: A = d 2^s = min(max(fma(l 2^-24, m, c), -x 2^s), (1-x) 2^s)
  uint32_t cm2, cc2;                         // fp16x2 m = step 2^(24+s), c = origin 2^s
  const uint4* clampc;                       // [n_base][ceil(n0/8)][2] {-x 2^s} | {(1-x) 2^s} fp16x2 words
  uint32_t rk[20];                           // Philox round keys of pert.seed
  float offlo, offhi;                        // PHILOX_CLAMP: smallest / largest offset * 2^s
};

struct alignas(16) Smem {
  uint64_t g_full[kSG], g_empty[kSG], w_full[kSW], w_empty[kSW];
  uint64_t acc1_full, acc2_full, acc3_full, acc2_free;
  uint64_t h1_pc[2 * kNkb2];                 // E1 pieces (32 neurons) handed to layer 2
  uint64_t h2_kb[kNkb2];
  uint32_t tbase;
  int base_e;
  // epilogue team: base data
  alignas(16) float ub1[kN1];
  alignas(16) float b1[kN1];                 // base1 of the staged base input (PHILOX_BOX)
  uint32_t nb1[8];
  float minub1;
  alignas(16) float ub2[kN2];
  alignas(16) float ub3[kN3P];
  alignas(16) float b3[kN3P];
  uint32_t nb2[8], nb3;
  float minub2, minub3;
  int bcls;
  // per-row partial results of the two halves of the epilogue team
  int xi[2][2][128];
  float xf[2][3][128];
  uint32_t sc2[8][128];                      // E2: sign-change words of layer 2
  uint16_t vc2[16][128];                     // E2 slow path: value-change bits of layer 2 (16 neurons)
  alignas(16) float c1row[8][kC1Rows][128];  // E2: the layer-2 potentials of a warp's few statistics rows
  alignas(16) uint4 ctab[kMaxN0 / 8][2];     // generators, PHILOX_CLAMP: the staged base's clamp bounds
  uint8_t stype[kMaxN0 / 64];                // ... and each stage's clamp type (kGen*)
};

constexpr size_t kTilesBytes = (size_t)(kSG + kSW) * kTile + (size_t)kChunks * kW3Chunk + 4 * kBiasTile;
constexpr size_t kSmemBytes = 1024 + kTilesBytes + sizeof(Smem);
static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");

struct TileInfo {
  int b;
  uint64_t start;     // first candidate index of the pair tile (range mode) or list position (eval)
  int nvalid;         // valid rows of the pair tile (0..256)
};

// The tile sequence of a cluster is contiguous, so (base, tile of the base) advance incrementally: one
// 64-bit division per thread per launch (TileIter's constructor), none per tile.
struct TileIter {
  int b;              // range mode: base input of the current tile
  uint64_t off;       // range mode: tile index inside the base's range
  __device__ __forceinline__ TileIter(const Args& a, uint64_t t0) {
    b = a.eval_idx ? a.eval_base : (int)(t0 / a.tiles_per_base);
    off = a.eval_idx ? t0 : t0 % a.tiles_per_base;
  }
  __device__ __forceinline__ void next(const Args& a) {
    if (++off == a.tiles_per_base && !a.eval_idx) { off = 0; b++; }
  }
  __device__ __forceinline__ TileInfo info(const Args& a) const {
    TileInfo ti;
    ti.b = b;
    if (a.eval_idx) {
      ti.start = off * 256;
      const int64_t rem = a.eval_n - (int64_t)ti.start;
      ti.nvalid = rem < 256 ? (int)rem : 256;
    } else {
      ti.start = a.pert.begin + off * 256;
      const uint64_t rem = a.pert.end - ti.start;
      ti.nvalid = rem < 256 ? (int)rem : 256;
    }
    return ti;
  }
};

// contiguous range of pair tiles owned by cluster c (base inputs change rarely inside a range)
__device__ __forceinline__ void cluster_range(uint64_t n, uint64_t c, uint64_t nc, uint64_t& t0, uint64_t& t1) {
  const uint64_t q = n / nc, r = n % nc;
  t0 = c * q + (c < r ? c : r);
  t1 = t0 + q + (c < r ? 1 : 0);
}

// Philox4x32-10 (reading C15) with the round keys of the launch's seed precomputed on the host
// (rk[2r], rk[2r+1] = key + r * Weyl): they stay in the parameter bank, so a round is two IMAD.WIDE
// and two LOP3 with a constant operand (no per-call key schedule).
__device__ __forceinline__ uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, const uint32_t (&rk)[20]) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ rk[2 * r], n2 = hi0 ^ c3 ^ rk[2 * r + 1];
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return make_uint4(c0, c1, c2, c3);
}
// The 8 levels of one Philox word (nibble n -> pixel n, LSB first) as the fp16 subnormals
// l * 2^-24, two per 32-bit word: one PRMT per pixel pair (the zero high bytes come from PRMT's
// sign replication of the nibble bytes).  The layer-1 MMA then computes 2^-24 * W1 l exactly in
// fp32 (products of an fp16 subnormal and an fp16 weight are exact; tools/test_subnormal_mma.py).
__device__ __forceinline__ uint4 nibble_word(uint32_t w) {
  const uint32_t lo = w & 0x0F0F0F0Fu;                   // nibbles 0, 2, 4, 6 in bytes 0..3
  const uint32_t hi = (w >> 4) & 0x0F0F0F0Fu;            // nibbles 1, 3, 5, 7
  uint32_t o[4];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const uint32_t sel = (uint32_t)k | ((8u + k) << 4) | ((4u + k) << 8) | ((12u + k) << 12);
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(o[k]) : "r"(lo), "r"(hi), "r"(sel));   // (__byte_perm drops
  }                                                                             //  the sign-replicate bit)
  return make_uint4(o[0], o[1], o[2], o[3]);
}

// PHILOX_CLAMP (reading C14): the A operand of a pixel pair, d 2^s = min(max(off 2^s, -x 2^s), (1-x) 2^s)
// in fp16, with off 2^s = fma(l 2^-24, step 2^(24+s), origin 2^s) from the subnormal levels.  Every
// step is exact (the host picked s so that each offset is an fp16 value; the bounds are exact where
// they bind, checked by the base prologue), so the layer-1 MMA contracts W1 (x' - x) exactly up to
// its fp32 accumulation of small terms.

// Stage clamp types (per base and 64-pixel stage, found when the base's bounds are staged): which
// bounds can bind anywhere in the stage.  kGenRelu: every pixel is 0, d = max(off, 0) = ReLU(off)
// (the FMA's .relu); kGenLower: only lower bounds bind, d = max(off, -x); kGenInterior: none, d = off;
// kGenGeneral: d = min(max(off, -x), 1 - x); kGenBox: PHILOX_BOX, A = the levels themselves.
constexpr int kGenRelu = 0, kGenLower = 1, kGenInterior = 2, kGenGeneral = 3, kGenBox = 4;
template <int TY>
__device__ __forceinline__ uint32_t gen_pair(uint32_t lv, uint32_t m2, uint32_t c2, uint32_t nx, uint32_t px) {
  if constexpr (TY == kGenBox) {
    return lv;
  } else if constexpr (TY == kGenRelu) {
    uint32_t d;
    asm("fma.rn.relu.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(lv), "r"(m2), "r"(c2));
    return d;
  } else {
    const __half2 o = __hfma2(*reinterpret_cast<const __half2*>(&lv), *reinterpret_cast<const __half2*>(&m2),
                              *reinterpret_cast<const __half2*>(&c2));
    if constexpr (TY == kGenInterior) return *reinterpret_cast<const uint32_t*>(&o);
    __half2 d = __hmax2(o, *reinterpret_cast<const __half2*>(&nx));
    if constexpr (TY == kGenGeneral) d = __hmin2(d, *reinterpret_cast<const __half2*>(&px));
    return *reinterpret_cast<const uint32_t*>(&d);
  }
}
// four pixel pairs (one 16-byte chunk of the A row) with the chunk's staged bounds {nx | px}
template <int TY>
__device__ __forceinline__ uint4 gen_chunk(uint4 o, const uint4 (&b)[2], uint32_t m2, uint32_t c2) {
  if constexpr (TY == kGenBox) return o;
  uint4 nx = make_uint4(0, 0, 0, 0), px = nx;
  if constexpr (TY == kGenLower || TY == kGenGeneral) nx = b[0];
  if constexpr (TY == kGenGeneral) px = b[1];
  return make_uint4(gen_pair<TY>(o.x, m2, c2, nx.x, px.x), gen_pair<TY>(o.y, m2, c2, nx.y, px.y),
                    gen_pair<TY>(o.z, m2, c2, nx.z, px.z), gen_pair<TY>(o.w, m2, c2, nx.w, px.w));
}

// h = max(u, 0) = hi + lo + O(2^-22 h): hi = RZ_f16(h), lo = RN_f16(h - hi) (relu'd), with the
// exact difference u - hi taken by one mixed-precision FMA (u + hi * -1).
__device__ __forceinline__ void split_pair(float u0, float u1, uint32_t& hi2, uint32_t& lo2) {
  asm("cvt.rz.relu.f16x2.f32 %0, %1, %2;" : "=r"(hi2) : "f"(u1), "f"(u0));
  float d0, d1;
  asm("{.reg .b16 l, h, m; mov.b16 m, 0xBC00; mov.b32 {l, h}, %2;\n\t"
      "fma.rn.f32.f16 %0, l, m, %3; fma.rn.f32.f16 %1, h, m, %4;}"
      : "=f"(d0), "=f"(d1) : "r"(hi2), "f"(u0), "f"(u1));
  asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(lo2) : "f"(d1), "f"(d0));
}

// sign bits of 32 potentials -> one word (bit i = neuron i): one funnel shift per neuron
__device__ __forceinline__ uint32_t sign_word(const uint32_t (&v)[32]) {
  uint32_t m = 0;
#pragma unroll
  for (int i = 31; i >= 0; i--) m = __funnelshift_l(v[i], m, 1);
  return m;
}
// sign bits of 16 potentials (bit i = neuron i) as two independent funnel-shift chains
__device__ __forceinline__ uint32_t sign16(const uint32_t (&v)[16]) {
  uint32_t a = 0, b = 0;
#pragma unroll
  for (int i = 7; i >= 0; i--) {
    a = __funnelshift_l(v[i], a, 1);
    b = __funnelshift_l(v[8 + i], b, 1);
  }
  return a | (b << 8);
}
// 3-input max / min (FMNMX3; |x| operands fold into the instruction)
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float min3f(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// acc = max(acc, |x_0| .. |x_15|) / min(acc, |x_0| .. |x_15|) as depth-3 trees
__device__ __forceinline__ float max_abs16(float acc, const float (&x)[16]) {
  const float m0 = max3f(fabsf(x[0]), fabsf(x[1]), fabsf(x[2])), m1 = max3f(fabsf(x[3]), fabsf(x[4]), fabsf(x[5]));
  const float m2 = max3f(fabsf(x[6]), fabsf(x[7]), fabsf(x[8])), m3 = max3f(fabsf(x[9]), fabsf(x[10]), fabsf(x[11]));
  const float m4 = max3f(fabsf(x[12]), fabsf(x[13]), fabsf(x[14]));
  return max3f(acc, max3f(m0, m1, m2), max3f(m3, m4, fabsf(x[15])));
}
__device__ __forceinline__ float min_abs16(float acc, const float (&x)[16]) {
  const float m0 = min3f(fabsf(x[0]), fabsf(x[1]), fabsf(x[2])), m1 = min3f(fabsf(x[3]), fabsf(x[4]), fabsf(x[5]));
  const float m2 = min3f(fabsf(x[6]), fabsf(x[7]), fabsf(x[8])), m3 = min3f(fabsf(x[9]), fabsf(x[10]), fabsf(x[11]));
  const float m4 = min3f(fabsf(x[12]), fabsf(x[13]), fabsf(x[14]));
  return min3f(acc, min3f(m0, m1, m2), min3f(m3, m4, fabsf(x[15])));
}
// sign bits of 16 potentials shifted into m from the top (bit i of the final word = neuron i when
// the upper half is folded first): one funnel shift per neuron
__device__ __forceinline__ uint32_t sign_fold(const uint32_t (&v)[16], uint32_t m) {
#pragma unroll
  for (int i = 15; i >= 0; i--) m = __funnelshift_l(v[i], m, 1);
  return m;
}

// layer-1 accumulators -> potentials: u1 = base1 + stepS * acc (reading C14b), in place
// (packed fp32 pairs: one FFMA2 per two neurons, the same single rounding as fmaf)
__device__ __forceinline__ void ffma2(uint32_t& x0, uint32_t& x1, uint64_t s2, float b0, float b1) {
  uint64_t d;
  const uint64_t x = (uint64_t)x0 | ((uint64_t)x1 << 32);
  const uint64_t b = (uint64_t)__float_as_uint(b0) | ((uint64_t)__float_as_uint(b1) << 32);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(s2), "l"(b));
  x0 = (uint32_t)d;
  x1 = (uint32_t)(d >> 32);
}
template <int N>
__device__ __forceinline__ void acc_to_u1(uint32_t (&v)[N], const float* b1, float stepS) {
  const float4* b4 = reinterpret_cast<const float4*>(b1);
  const uint64_t s2 = (uint64_t)__float_as_uint(stepS) * 0x100000001ull;
#pragma unroll
  for (int k = 0; k < N / 4; k++) {
    const float4 bb = b4[k];
    ffma2(v[4 * k], v[4 * k + 1], s2, bb.x, bb.y);
    ffma2(v[4 * k + 2], v[4 * k + 3], s2, bb.z, bb.w);
  }
}
// sign bits of 32 potentials as four independent funnel-shift chains (bit i = neuron i)
__device__ __forceinline__ uint32_t sign32(const uint32_t (&v)[32]) {
  uint32_t a = 0, b = 0, c = 0, d = 0;
#pragma unroll
  for (int i = 7; i >= 0; i--) {
    a = __funnelshift_l(v[i], a, 1);
    b = __funnelshift_l(v[8 + i], b, 1);
    c = __funnelshift_l(v[16 + i], c, 1);
    d = __funnelshift_l(v[24 + i], d, 1);
  }
  return a | (b << 8) | (c << 16) | (d << 24);
}
// the two epilogue warps of a TMEM lane quadrant (halves h = 0, 1 of the neurons, same rows) combine
// their per-row partial results through shared memory (named barrier `id`, 64 threads)
__device__ __forceinline__ void pair_exchange_i(Smem& S, int h, int r, int& nsc, int& istar, int id) {
  S.xi[h][0][r] = nsc;
  S.xi[h][1][r] = istar;
  named_bar(id, 64);
  const int o = h ^ 1, onsc = S.xi[o][0][r], oist = S.xi[o][1][r];
  nsc += onsc;
  if (oist >= 0 && (istar < 0 || oist < istar)) istar = oist;   // lowest changed neuron of the row
  named_bar(id, 64);                                      // the slots are reused by the next exchange
}
__device__ __forceinline__ void pair_exchange_f(Smem& S, int h, int r, float& mx, float& mn, float& mn2, int id) {
  S.xf[h][0][r] = mx;
  S.xf[h][1][r] = mn;
  S.xf[h][2][r] = mn2;
  named_bar(id, 64);
  const int o = h ^ 1;
  mx = fmaxf(mx, S.xf[o][0][r]);
  mn = fminf(mn, S.xf[o][1][r]);
  mn2 = fminf(mn2, S.xf[o][2][r]);
  named_bar(id, 64);
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
  uint8_t* sW3 = sW + kSW * kTile;                       // [kChunks][1 KB] W3 half (resident)
  uint8_t* sOnes = sW3 + kChunks * kW3Chunk;             // [4 KB] ones column (bias MMA A)
  uint8_t* sB2 = sOnes + kBiasTile;                      // [4 KB] [b2_hi | b2_lo] half (bias MMA B)
  uint8_t* sT = sB2 + kBiasTile;                         // [2][4 KB] h2 hi / lo of neurons 240-255
  Smem& S = *reinterpret_cast<Smem*>(sT + 2 * kBiasTile);

  const uint32_t rank = cluster_ctarank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  uint64_t t_begin, t_end;
  cluster_range(a.n_pairs_tiles, cluster, nclusters, t_begin, t_end);

  if (threadIdx.x == 0) {
    const uint32_t two = rank == 0 ? 2u : 1u;
    for (int i = 0; i < kSG; i++) { mbar_init(&S.g_full[i], 8); mbar_init(&S.g_empty[i], 1); }
    for (int i = 0; i < kSW; i++) { mbar_init(&S.w_full[i], two); mbar_init(&S.w_empty[i], 1); }
    mbar_init(&S.acc1_full, 1); mbar_init(&S.acc2_full, 1); mbar_init(&S.acc3_full, 1);
    mbar_init(&S.acc2_free, 8);
    for (int i = 0; i < 2 * kNkb2; i++) mbar_init(&S.h1_pc[i], 8);    // 4 warps x 2 CTAs
    for (int i = 0; i < kNkb2; i++) mbar_init(&S.h2_kb[i], i ? 8 : 16);   // block 0 also waits for group 15's read
    S.base_e = -1;
    fence_mbar_init();
  }
  if (warp == kWIss) { tmem_alloc2(&S.tbase, 512); tmem_relinquish2(); }
  // resident operands: W3 half, ones column, bias-2 half (plain 16-byte copies, once)
  {
    const uint4* s3 = reinterpret_cast<const uint4*>(a.wblk + a.lay.w3 + (size_t)rank * kChunks * kW3Chunk);
    uint4* d3 = reinterpret_cast<uint4*>(sW3);
    for (int i = threadIdx.x; i < (int)(kChunks * kW3Chunk / 16); i += kThreads) d3[i] = s3[i];
    const uint4* so = reinterpret_cast<const uint4*>(a.wblk + a.lay.ones);
    const uint4* sb = reinterpret_cast<const uint4*>(a.wblk + a.lay.bias2 + (size_t)rank * kBiasTile);
    uint4* dO = reinterpret_cast<uint4*>(sOnes);
    uint4* dB = reinterpret_cast<uint4*>(sB2);
    for (int i = threadIdx.x; i < (int)(kBiasTile / 16); i += kThreads) { dO[i] = so[i]; dB[i] = sb[i]; }
  }
  fence_proxy_async();
  fence_before();
  cluster_sync();
  fence_after();
  const uint32_t tb = S.tbase;
  const uint32_t R1 = tb, R2 = tb + 256u, R3 = tb + 496u;
  const int nst = a.lay.nst;

  // (each branch starts with its warpgroups' setmaxnreg, so that ptxas allocates per role)
  if (warp < kWE || warp >= kWE + 8) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegGen));
  if (warp >= kWE + 8) {
  if (warp == kWProd) {
    // ------------------------------------------------------------------ weight producer (both CTAs)
    if (lane == 0) {
      uint32_t ws = 0;
      const uint8_t* src0 = a.wblk + a.lay.stream + (size_t)rank * nst * kTile;
      for (uint64_t t = t_begin; t < t_end; t++)
        for (int s = 0; s < nst; s++) {
          const uint32_t st = ws % kSW, ph = (ws / kSW) & 1u;
          mbar_wait_sleep(&S.w_empty[st], ph ^ 1u, 128);
#if MLPV_EXP == 104
          if (t == t_begin) {
            mbar_expect_tx(&S.w_full[st], kTile);
            bulk_g2s(sW + st * kTile, src0 + (size_t)s * kTile, kTile, &S.w_full[st]);
          } else mbar_arrive(&S.w_full[st]);
#else
          mbar_expect_tx(&S.w_full[st], kTile);
          bulk_g2s(sW + st * kTile, src0 + (size_t)s * kTile, kTile, &S.w_full[st]);
#endif
          ws++;
        }
    }
  } else if (warp == kWIss) {
    if (lane == 0 && rank == 1) {
      // ---------------------------------------------------------------- peer: relay its weight stages
      uint32_t ws = 0;
      for (uint64_t t = t_begin; t < t_end; t++)
        for (int s = 0; s < nst; s++) {
          const uint32_t st = ws % kSW, ph = (ws / kSW) & 1u;
          mbar_wait(&S.w_full[st], ph);
          mbar_arrive_cluster(&S.w_full[st], 0);
          ws++;
        }
    } else if (rank == 0) {
      // ---------------------------------------------------------------- MMA issuer (leader)
      // The tensor pipe takes a new MMA only about when the previous one is under way, so every
      // cycle this thread spends between two MMAs is a pipe bubble: the waits for stage s+1 are
      // placed after the second MMA of stage s, and the commits that free stage s's ring slots
      // after the first MMA of stage s+1 (never across the layer-1 -> layer-2 boundary, which
      // depends on E1 and so on this tile's own layer-1 MMAs).  The whole warp runs the loop
      // (warp-uniform descriptors in uniform registers); one elected lane issues.
      const bool el = elect_one();
      const uint32_t id1 = idesc_f16(256, kN1, 0, 0);     // f16 levels x f16 W1 -> f32
      const uint32_t id2 = idesc_f16(256, kN2, 0, 0);     // f16 x f16 -> f32
      uint32_t gslot = 0, gph = 0, wslot = 0, wph = 0;    // ring position of the next stage
      int pend_g = -1, pend_w = -1;                       // slots of the previous stage, not yet committed
      auto flush = [&]() {
        if (el && pend_g >= 0) mma2_commit(&S.g_empty[pend_g], 0x3);
        if (el && pend_w >= 0) mma2_commit(&S.w_empty[pend_w], 0x3);
        pend_g = pend_w = -1;
      };
      auto wait_l1 = [&]() {
        mbar_wait(&S.g_full[gslot], gph);
        mbar_wait(&S.w_full[wslot], wph);
      };
      const uint32_t aLo0 = sdesc_sw128_lo(smem_u32(sG)), bLo0 = sdesc_sw128_lo(smem_u32(sW));
      const int nk_last = a.nk16 - 4 * (a.nkb1 - 1);      // K16 steps of the last layer-1 stage (1..4)
      // Layer 3 of the previous tile is issued from here too, one 64-neuron block (8 small MMAs)
      // at a time as E2 hands the blocks over, between layer-1 stages: a second issuing warp would
      // queue its MMAs behind the whole layer-1 backlog of the tensor pipe (and E3 -- hence E1 of
      // the next tile -- would wait for them).
      const uint32_t id3 = idesc_f16(256, kN3P, 0, 0);
      int l3_kb = kNkb2;                                  // next layer-3 block of tile l3_tl (kNkb2: none)
      uint32_t l3_tl = 0;
      auto issue_l3 = [&]() {                             // elected lane: block l3_kb of tile l3_tl
#pragma unroll
        for (int kk = 0; kk < 4; kk++) {
          if (MLPV_EXP == 105) break;
          const int g = 4 * l3_kb + kk;
          const uint64_t bd = sdesc_sw128(smem_u32(sW3 + (g >> 1) * kW3Chunk) + 32u * (g & 1));
          if (g < 15) {
            mma2_f16_ts(R3, R2 + 16u * g, bd, id3, g ? 1u : 0u);
            mma2_f16_ts(R3, R2 + 16u * g + 8u, bd, id3, 1u);
          } else {
            mma2_f16_ss(R3, sdesc_none(smem_u32(sT), 128, 256), bd, id3, 1u);
            mma2_f16_ss(R3, sdesc_none(smem_u32(sT + kBiasTile), 128, 256), bd, id3, 1u);
          }
        }
        if (l3_kb == 0) TR(l3_tl, 14);
        if (l3_kb == kNkb2 - 1) { mma2_commit(&S.acc3_full, 0x3); TR(l3_tl, 15); }
      };
      auto drain_l3 = [&]() {                             // the rest of layer 3, blocking
        while (l3_kb < kNkb2) {
          mbar_wait_sleep(&S.h2_kb[l3_kb], l3_tl & 1u, 32);
          fence_after();
          if (el) issue_l3();
          l3_kb++;
        }
      };
      uint32_t tl = 0;
      if (t_begin < t_end) wait_l1();
      for (uint64_t t = t_begin; t < t_end; t++, tl++) {
        TR(tl, 0);
        // layer 1 into R1 (issued after the previous tile's layer 2, which read R1: in-order pipe).
        // Lean loop: the issuing warp runs one dependent instruction chain, so every instruction
        // between two MMAs shows up in the stage time (descriptors are low words + immediates).
        for (int kb = 0; kb < a.nkb1; kb++) {
          TRI(tl, kb, 0);
          fence_after();
          const uint32_t alo = aLo0 + (uint32_t)gslot * (kTile >> 4), blo = bLo0 + (uint32_t)wslot * (kTile >> 4);
          const int cg = (int)gslot, cw = (int)wslot;
          if (++gslot == kSG) { gslot = 0; gph ^= 1u; }
          if (++wslot == kSW) { wslot = 0; wph ^= 1u; }
          const bool full = kb + 1 < a.nkb1;                 // all four K16 steps (the last stage: nk_last)
          // the elected lane tests the next stage first and reads the answers after this stage's MMAs
          // (same basic block, so the SYNCS round trip overlaps the issue)
          uint32_t notready = 0, l3go = 0;
          if (el) {
            const bool r1 = mbar_test(&S.g_full[gslot], gph), r2 = mbar_test(&S.w_full[wslot], wph);
            const bool r3 = l3_kb < kNkb2 && mbar_test(&S.h2_kb[l3_kb & 3], l3_tl & 1u);
            mma2_f16_ss_lo(R1, alo, blo, id1, kb ? 1u : 0u);
            TRI(tl, kb, 2);
            if (pend_g >= 0) mma2_commit(&S.g_empty[pend_g], 0x3);
            if (pend_w >= 0) mma2_commit(&S.w_empty[pend_w], 0x3);
            TRI(tl, kb, 4);
            if (full || nk_last > 1) mma2_f16_ss_lo(R1, alo + 2u, blo + 2u, id1, 1u);
            TRI(tl, kb, 5);
            if (full || nk_last > 2) mma2_f16_ss_lo(R1, alo + 4u, blo + 4u, id1, 1u);
            TRI(tl, kb, 6);
            if (full || nk_last > 3) mma2_f16_ss_lo(R1, alo + 6u, blo + 6u, id1, 1u);
            TRI(tl, kb, 7);
            notready = (r1 && r2) ? 0u : 1u;
            if (r3) {
              fence_after();
              issue_l3();
              l3go = 1u;
            }
          }
          if (__any_sync(0xffffffffu, l3go)) l3_kb++;
          pend_g = cg; pend_w = cw;
          if (full && __any_sync(0xffffffffu, notready)) {
            // wait for the next stage; meanwhile issue whatever layer-3 block E2 has handed over
            // (the pipe would otherwise hold L3 -- and so E3, and the next E1 -- behind a
            // generator-bound layer 1)
            TRI(tl, kb, 1);
            bool d1 = false, d2 = false;
            while (true) {
              if (!d1) d1 = mbar_try_ns(&S.g_full[gslot], gph, 200u);
              if (!d2) d2 = mbar_test(&S.w_full[wslot], wph);
              if (__all_sync(0xffffffffu, d1 && d2)) break;
              if (l3_kb < kNkb2 && __all_sync(0xffffffffu, mbar_test(&S.h2_kb[l3_kb & 3], l3_tl & 1u))) {
                fence_after();
                if (el) issue_l3();
                l3_kb++;
              }
            }
            TRI(tl, kb, 3);
          }
        }
        flush();
        if (el) mma2_commit(&S.acc1_full, 0x3);
        TR(tl, 2);
        drain_l3();                                         // E3 of the previous tile frees R2
        // layer 2: D = R2 <- bias (ones x [b_hi | b_lo]) + H1 (fp16 hi | lo, TMEM) x W2 half tiles
        mbar_wait_sleep(&S.acc2_free, (tl & 1u) ^ 1u, 64);
        TR(tl, 4);
        fence_after();                                      // the bias needs only R2, not H1
        if (el) mma2_f16_ss(R2, sdesc_none(smem_u32(sOnes), 128, 256), sdesc_none(smem_u32(sB2), 128, 256), id2, 0u);
        mbar_wait_sleep(&S.h1_pc[0], tl & 1u, 32);
        TR(tl, 3);
        mbar_wait(&S.w_full[wslot], wph);
        for (int kb = 0; kb < kNkb2; kb++) {
          fence_after();
          const uint32_t bb = smem_u32(sW + wslot * kTile);
          const int cw = (int)wslot;
          if (++wslot == kSW) { wslot = 0; wph ^= 1u; }
#pragma unroll
          for (int kk = 0; kk < 4; kk++) {
            const uint32_t col = 16u * (4u * kb + kk);      // neurons [col, col+16): hi | lo
            const uint64_t bd = sdesc_sw128(bb + 32u * kk);
            if (el) {
              mma2_f16_ts(R2, R1 + col, bd, id2, 1u);
              mma2_f16_ts(R2, R1 + col + 8u, bd, id2, 1u);
            }
            if (kk == 0) flush();
            // H1 arrives in 32-neuron pieces (K steps 2 per piece): wait for each piece just before
            // its K steps, so layer 2 starts one piece after E1 does
            if (kk == 1) mbar_wait_sleep(&S.h1_pc[2 * kb + 1], tl & 1u, 32);
            if (kk == 3) {
              if (kb + 1 < kNkb2) {
                mbar_wait_sleep(&S.h1_pc[2 * kb + 2], tl & 1u, 32);
                mbar_wait(&S.w_full[wslot], wph);
              } else if (t + 1 < t_end) {
                wait_l1();                                  // the next tile's first layer-1 stage
              }
            }
          }
          pend_w = cw;
        }
        if (el) mma2_commit(&S.acc2_full, 0x3);
        TR(tl, 5);
        l3_tl = tl; l3_kb = 0;                              // this tile's layer 3 follows E2
      }
      flush();
      drain_l3();
    }
#ifdef MLPV_TRACE
  } else if (warp == kWIdle) {
    if (lane == 0 && rank == 0 && cluster == 0) {
      uint32_t gs = 0;
      for (uint64_t t = t_begin; t < t_end && gs < 12u * (uint32_t)a.nkb1; t++)
        for (int kb = 0; kb < a.nkb1; kb++, gs++) {
          mbar_wait(&S.g_empty[gs % kSG], (gs / kSG) & 1u);
          const uint32_t tl = gs / (uint32_t)a.nkb1;
          if (tl >= 8 && tl < 12) g_trace_done[tl - 8][kb] = clock64();
        }
    }
#endif
  }
  } else {
    // ------------------------------------------------------------------ generator (both CTAs)
    // Three groups of four warps take the ring stages in turn; a warp generates a whole 64-pixel K
    // block of its 32 rows (two Philox calls) into registers before it waits for the slot.  The A
    // operand is the level l of every pixel (reading C14b: x' = x + origin + l * step, linear in l);
    // the base image enters through base1 in the epilogue.
    if ((gen_index(warp) >> 2) < kNGenGroups) {          // (MLPV_EXP 31: fewer generator groups)
    const int gw = gen_index(warp), grp = gw >> 2;
    const int r = 32 * (gw & 3) + lane;                    // row of this CTA's A tile
    const int gt = 32 * gw + lane;                         // 0..383
    uint32_t tl = 0;
    const int nblk = (a.n0 + 31) / 32;                     // Philox blocks holding pixels
    const bool clampk = a.clamp != 0;
    int gbase = -1;                                        // base whose clamp bounds are staged
    TileIter tit(a, t_begin);
    for (uint64_t t = t_begin; t < t_end; t++, tl++, tit.next(a)) {
      if (gt == 0) TR(tl, 6);
      const TileInfo ti = tit.info(a);
      if (clampk && ti.b != gbase) {
        // every generator thread meets this barrier at the same tile (the tile sequence is the
        // cluster's), after all its stages of the previous base: then the table is free
        named_bar(13, 32 * kNGenGroups * 4);
        const int nch = (a.n0 + 7) / 8;
        const uint4* src = a.clampc + (size_t)ti.b * 2 * nch;
        for (int i = gt; i < 2 * (kMaxN0 / 8); i += 32 * kNGenGroups * 4)
          (&S.ctab[0][0])[i] = (i >> 1) < nch ? src[i] : make_uint4(0, 0, 0, 0);   // beyond n_0: d = 0
        named_bar(13, 32 * kNGenGroups * 4);
        if (gt < kMaxN0 / 64) {
          // the stage's type from its 64 pixels' bounds (padding pixels, nx = px = +0, constrain nothing)
          bool lower = false, upper = false, zero = true;
          for (int ch = 0; ch < 8; ch++)
            for (int w = 0; w < 4; w++) {
              const uint32_t nx2 = (&S.ctab[8 * gt + ch][0].x)[w], px2 = (&S.ctab[8 * gt + ch][1].x)[w];
              for (int hh = 0; hh < 2; hh++) {
                const uint16_t nb = (uint16_t)(nx2 >> (16 * hh)), pb = (uint16_t)(px2 >> (16 * hh));
                if (nb == 0 && pb == 0) continue;
                const float nx = __half2float(__ushort_as_half(nb)), px = __half2float(__ushort_as_half(pb));
                if (nx > a.offlo) lower = true;
                if (px < a.offhi) upper = true;
                if (nb != 0x8000u) zero = false;
              }
            }
          S.stype[gt] = (uint8_t)(upper ? kGenGeneral : (lower ? (zero ? kGenRelu : kGenLower) : kGenInterior));
        }
        named_bar(13, 32 * kNGenGroups * 4);
        gbase = ti.b;
      }
      const int grow = 128 * (int)rank + r;
      uint64_t c;
      if (a.eval_idx) c = grow < ti.nvalid ? a.eval_idx[ti.start + grow] : 0;
      else c = ti.start + (uint64_t)grow;
      const uint32_t c0 = (uint32_t)c, c1 = (uint32_t)(c >> 32), cb = (uint32_t)ti.b;
#if MLPV_EXP != 108
      const PhiloxRow prow = philox_row(c0, c1, cb, a.rk);
#endif
      const uint32_t gs0 = tl * (uint32_t)a.nkb1;          // global index of this tile's first stage
      for (int kb = (int)((grp + kNGenGroups - gs0 % kNGenGroups) % kNGenGroups); kb < a.nkb1; kb += kNGenGroups) {
        const uint32_t gs = gs0 + kb;
        // one stage, specialised on its clamp type (uniform per stage; see gen_chunk)
        auto stage = [&](auto tyc) {
          constexpr int TY = decltype(tyc)::value;
          TRG(tl, kb, 0);
          // A operand of the 64-pixel K block: the first 32 pixels (Philox block 2 kb) are finished
          // before the slot wait, the second block's words stay raw (4 registers) until after it
          // (the clamped form would not fit the generator's 72 registers with all 8 chunks live)
          uint4 out[4];
          uint4 w1;
          {
            const int j = 2 * kb;
            const uint4 z = make_uint4(0, 0, 0, 0);
#if MLPV_EXP == 108
            const uint4 w0 = make_uint4(c0 * 0x9E3779B9u + j, c0 ^ (uint32_t)j, c0 + 77u * j, c0 * 3u), z2 = z;
            w1 = make_uint4(c0 * 0x85EBCA6Bu + j, c0 ^ (uint32_t)(j * 9), c0 + 33u * j, c0 * 5u + z2.x);
#else
            const uint4 w0 = j < nblk ? philox_j(prow, (uint32_t)j, a.rk) : z;
            w1 = j + 1 < nblk ? philox_j(prow, (uint32_t)(j + 1), a.rk) : z;
#endif
            out[0] = nibble_word(w0.x); out[1] = nibble_word(w0.y);
            out[2] = nibble_word(w0.z); out[3] = nibble_word(w0.w);
#pragma unroll
            for (int ch = 0; ch < 4; ch++) out[ch] = gen_chunk<TY>(out[ch], S.ctab[8 * kb + ch], a.cm2, a.cc2);
          }
          const uint32_t st = gs % kSG, ph = (gs / kSG) & 1u;
          TRG(tl, kb, 1);
          if ((gw & 3) == 0) mbar_wait_sleep(&S.g_empty[st], ph ^ 1u, MLPV_F3_GEN_SLEEP);   // one poller per group
          named_bar(6 + grp, 128);
          TRG(tl, kb, 2);
          uint8_t* slot = sG + st * kTile;
#pragma unroll
          for (int ch = 0; ch < 4; ch++)                       // (K steps beyond nk16 are written too: the
            if (MLPV_EXP != 21)                                //  MMA never reads them, the slot holds 64)
              *reinterpret_cast<uint4*>(slot + sw128_off(r, 16 * ch)) = out[ch];
          const uint32_t w1w[4] = {w1.x, w1.y, w1.z, w1.w};
#pragma unroll
          for (int ch = 4; ch < 8; ch++) {
            const uint4 o = gen_chunk<TY>(nibble_word(w1w[ch - 4]), S.ctab[8 * kb + ch], a.cm2, a.cc2);
            if (MLPV_EXP != 21)
              *reinterpret_cast<uint4*>(slot + sw128_off(r, 16 * ch)) = o;
          }
          fence_proxy_async();
          __syncwarp();
          TRG(tl, kb, 3);
          if (lane == 0) arrive_leader(&S.g_full[st], rank);
        };
        switch (clampk ? (int)S.stype[kb] : kGenBox) {
          case kGenRelu: stage(std::integral_constant<int, kGenRelu>{}); break;
          case kGenLower: stage(std::integral_constant<int, kGenLower>{}); break;
          case kGenInterior: stage(std::integral_constant<int, kGenInterior>{}); break;
          case kGenBox: stage(std::integral_constant<int, kGenBox>{}); break;
          default: stage(std::integral_constant<int, kGenGeneral>{}); break;
        }
        TRG(tl, kb, 4);
      }
      if (gt == 0) TR(tl, 7);
    }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegEpi));
    // ------------------------------------------------------------------ epilogue team (E1, E2, E3)
    // Eight warps, two per TMEM lane quadrant (halves h = 0, 1; same rows, different neurons).  Half
    // 0 runs E1(t) -> E2(t) -> E1(t+1), half 1 E1(t) -> E2(t) -> E3(t) -> E1(t+1): the order in which
    // the accumulators become ready (E2(t) overlaps the layer-1 MMAs of tile t+1).  Per-row partial
    // results of the two halves meet in shared memory.
    const int q = warp & 3, h = (warp - kWE) >> 2;
    const int r = 32 * q + lane;                           // row = TMEM lane
    const int et = threadIdx.x - 32 * kWE;                 // 0..255
    const uint32_t loff = (uint32_t)(32 * q) << 16;
    const float th1 = a.cov.th_f[0], tg2 = a.cov.tg_f[1], tg3 = a.cov.tg_f[2], th2 = a.cov.th_f[1];
    const float tau0 = a.cov.tau_dev ? a.cov.tau_dev[0] : a.cov.tau[0];
    const float tau1 = a.cov.tau_dev ? a.cov.tau_dev[1] : a.cov.tau[1];
    const float tau2 = a.cov.tau_dev ? a.cov.tau_dev[2] : a.cov.tau[2];
    const bool eval = a.eval_idx != nullptr;
    const bool need12 = a.pair12 >= 0 && !eval, need23 = a.pair23 >= 0 && !eval;
    const float stepS = a.stepS;
    const bool clampk = a.clamp != 0;
    uint32_t tl = 0;
    TileIter tit(a, t_begin);
    for (uint64_t t = t_begin; t < t_end; t++, tl++, tit.next(a)) {
      const TileInfo ti = tit.info(a);
      const int grow = 128 * (int)rank + r;
      // a row outside the restriction R (Philox spaces, k_restrict_mask) gets no verdict / coverage
      const bool valid = grow < ti.nvalid && (eval || in_restriction(a.pert, ti.b, ti.start + (uint64_t)grow));
      const uint64_t cidx = eval ? (uint64_t)(ti.start + grow) : 0;
      if (ti.b != S.base_e) {                              // stage the base traces once per base input
        named_bar(2, 256);
        const float* tr = a.trace + (size_t)ti.b * a.T;
        for (int i = et; i < kN1; i += 256) {
          S.ub1[i] = tr[i];
          S.b1[i] = a.base1[(size_t)ti.b * kN1 + i];
        }
        for (int i = et; i < kN2; i += 256) S.ub2[i] = tr[kN1 + i];
        if (et < kN3P) {
          S.ub3[et] = et < a.n3 ? tr[kN1 + kN2 + et] : 0.f;
          S.b3[et] = et < a.n3 ? a.b3[et] : 0.f;
        }
        named_bar(2, 256);
        if (et < 8) {
          uint32_t m = 0;
          for (int i = 0; i < 32; i++) m |= (__float_as_uint(S.ub1[32 * et + i]) >> 31) << i;
          S.nb1[et] = m;
        } else if (et < 16) {
          uint32_t m = 0;
          for (int i = 0; i < 32; i++) m |= (__float_as_uint(S.ub2[32 * (et - 8) + i]) >> 31) << i;
          S.nb2[et - 8] = m;
        } else if (et == 16) {
          uint32_t m = 0;
          for (int i = 0; i < a.n3; i++) m |= (__float_as_uint(S.ub3[i]) >> 31) << i;
          S.nb3 = m;
        } else if (et == 17) {
          float m = 3.0e38f;
          for (int i = 0; i < kN1; i++) m = fminf(m, fabsf(S.ub1[i]));
          S.minub1 = m;
        } else if (et == 18) {
          float m = 3.0e38f;
          for (int i = 0; i < kN2; i++) m = fminf(m, fabsf(S.ub2[i]));
          S.minub2 = m;
        } else if (et == 19) {
          float m = 3.0e38f;
          for (int i = 0; i < a.n3; i++) m = fminf(m, fabsf(S.ub3[i]));
          S.minub3 = m;
          S.bcls = a.cls[ti.b];
        }
        named_bar(2, 256);
        if (et == 0) S.base_e = ti.b;
      }
      // =========================== E1: layer-1 potentials -> predicates, H1 = fp16 hi | lo in place
      // (one warp polls; the others sleep in bar.sync)
      // each half waits on its own (half 1 comes from the previous tile's E3)
      if ((et & 127) == 0) { mbar_wait_sleep(&S.acc1_full, tl & 1u, 64); }
      named_bar(h ? 14 : 3, 128);
      if (et == 0) TR(tl, 8);
      TRE(0, tl, 0);
      TRE2(tl, 0, 0);
      fence_after();
      // single pass, one piece (32 neurons = 32 columns) per step; half h takes pieces h, h+2, h+4,
      // h+6, so both halves contribute to every 64-neuron block and block k is handed to the MMA
      // after step k of each half.  Per piece: u1 = base1 + stepS * acc (reading C14b), H1 = fp16
      // hi | lo in place (one 32-column store), sign-change bits, and L-inf / min |u| while some row
      // of the warp can still end with <= 1 change.  32 columns per step give the scheduler two
      // independent 16-neuron chains (the step is latency-bound).
      int nsc1 = 0, istar1 = -1;
      float linf1 = 0.f, minab1 = 3.0e38f;
#pragma unroll 1
      for (int k4 = 0; k4 < (h ? 3 : 5); k4++) {
        // half 0: pieces 0, 1, 2, 4, 6 (block 0 alone); half 1, which first finishes the previous
        // tile's E3: pieces 3, 5, 7
        const int p = h ? 2 * k4 + 3 : (k4 < 2 ? k4 : 2 * k4 - 2);   // piece: groups 2p, 2p + 1
        const int kbs = p >> 1;                            // the 64-neuron block it completes a part of
        uint32_t v[32];
        TR1(tl, k4, 0);
        tmem_ld32(R1 + loff + 32u * p, v);
        tmem_ld_wait();
        TR1(tl, k4, 1);
        // statistics wanted while some row of the warp can still end with <= 1 change (below)
        const bool stat1 = __any_sync(0xffffffffu, need12 && valid && nsc1 <= 1);
        if (stat1 && clampk) {
          // PHILOX_CLAMP: u1 - u1_base = 2^-s acc exactly up to the accumulation (the base trace is
          // base1), so the L-inf partial is max |acc| (scaled by 2^-s once, after the pass)
          float aa[16], ab[16];
#pragma unroll
          for (int j = 0; j < 16; j++) { aa[j] = __uint_as_float(v[j]); ab[j] = __uint_as_float(v[16 + j]); }
          linf1 = max_abs16(max_abs16(linf1, aa), ab);
        }
        acc_to_u1(v, S.b1 + 32 * p, stepS);
        uint32_t hl[32];                                   // [hi 2p | lo 2p | hi 2p+1 | lo 2p+1]
#pragma unroll
        for (int k = 0; k < 8; k++) {
          split_pair(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]), hl[k], hl[8 + k]);
          split_pair(__uint_as_float(v[16 + 2 * k]), __uint_as_float(v[16 + 2 * k + 1]), hl[16 + k], hl[24 + k]);
        }
        tmem_st32(R1 + loff + 32u * p, hl);
        const uint32_t s = sign32(v) ^ S.nb1[p];
        nsc1 += __popc(s);
        if (istar1 < 0 && s) istar1 = 32 * p + __ffs(s) - 1;
        if (eval && valid) {
#pragma unroll
          for (int j = 0; j < 32; j++) a.eval_out[cidx * a.T + 32 * p + j] = __uint_as_float(v[j]);
        }
        if (stat1 && clampk) {
          float u0[16], u1v[16];
#pragma unroll
          for (int j = 0; j < 16; j++) { u0[j] = __uint_as_float(v[j]); u1v[j] = __uint_as_float(v[16 + j]); }
          minab1 = min_abs16(min_abs16(minab1, u0), u1v);
        } else if (stat1) {
#pragma unroll
          for (int hh = 0; hh < 2; hh++) {
            const float4* ub = reinterpret_cast<const float4*>(S.ub1 + 32 * p + 16 * hh);
            float uu[16], d[16];
#pragma unroll
            for (int k = 0; k < 4; k++) {
              const float4 b4 = ub[k];
              const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
              for (int j = 0; j < 4; j++) {
                uu[4 * k + j] = __uint_as_float(v[16 * hh + 4 * k + j]);
                d[4 * k + j] = uu[4 * k + j] - bb[j];
              }
            }
            linf1 = max_abs16(linf1, d);
            minab1 = min_abs16(minab1, uu);
          }
        }
        TR1(tl, k4, 2);
        {                                                  // every piece signs off its half of the block
          tmem_st_wait();
          fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(&S.h1_pc[p], rank);
          TRE(0, tl, 2 + kbs);
          TRE2(tl, 0, 2 + kbs);
        }
        TR1(tl, k4, 3);
      }
      TRE(0, tl, 1);
      pair_exchange_i(S, h, r, nsc1, istar1, 9 + q);
      TRE2(tl, 0, 6);
      // only a candidate with at most one sign change in layer 1 can fire a covering method on pair
      // (1, 2); for those rows both halves computed their L-inf / min |u| partials above
      const bool slow1 = __any_sync(0xffffffffu, need12 && valid && nsc1 <= 1);
      float dummy = 0.f;
      if (slow1) pair_exchange_f(S, h, r, linf1, minab1, dummy, 9 + q);
      if (clampk) linf1 *= stepS;                         // max |acc| -> max |u1 - u1_base|
      minab1 = fminf(minab1, S.minub1);
      const bool cond1 = need12 && valid && ((nsc1 == 1) || (nsc1 == 0 && linf1 >= th1));
      const bool amb1 = minab1 < tau0 || (nsc1 == 0 && fabsf(linf1 - th1) < tau0);
      if (et == 0) TR(tl, 9);
      // =========================== E2: layer-2 potentials -> predicates, H2 (hi | lo) for layer 3
      if (et == 0) { mbar_wait_sleep(&S.acc2_full, tl & 1u, 64); }
      named_bar(4, 256);
      if (et == 0) TR(tl, 10);
      TRE(1, tl, 0);
      TRE2(tl, 1, 0);
      fence_after();
      // pass A: sign-change words of layer 2 (kept in shared memory, row-private)
      int nsc2 = 0, istar2 = -1;
#pragma unroll 1
      for (int pp = 0; pp < 4; pp += 2) {
        const int p = 4 * h + pp;
        uint32_t va[32], vb[32];
#if MLPV_EXP == 106
#pragma unroll
        for (int j = 0; j < 32; j++) { va[j] = (uint32_t)j * lane; vb[j] = va[j] ^ 5u; }
#else
        tmem_ld32(R2 + loff + 32u * p, va);
        tmem_ld32(R2 + loff + 32u * p + 32u, vb);
        tmem_ld_wait();
#endif
        const uint32_t sa = sign32(va) ^ S.nb2[p], sb = sign32(vb) ^ S.nb2[p + 1];
        S.sc2[p][r] = sa;
        S.sc2[p + 1][r] = sb;
        nsc2 += __popc(sa) + __popc(sb);
        if (istar2 < 0 && sa) istar2 = 32 * p + __ffs(sa) - 1;
        if (istar2 < 0 && sb) istar2 = 32 * p + 32 + __ffs(sb) - 1;
        if (eval && valid) {
#pragma unroll
          for (int j = 0; j < 32; j++) {
            a.eval_out[cidx * a.T + kN1 + 32 * p + j] = __uint_as_float(va[j]);
            a.eval_out[cidx * a.T + kN1 + 32 * p + 32 + j] = __uint_as_float(vb[j]);
          }
        }
      }
      pair_exchange_i(S, h, r, nsc2, istar2, 9 + q);
      const bool slow2 = __any_sync(0xffffffffu, cond1 || (need23 && valid && nsc2 <= 1));
      // Layer-2 statistics (min |u|, L-inf, value-change words and their margin) are needed only
      // by rows with cond1 (pair (1, 2)) or with at most one layer-2 sign change (pair (2, 3)):
      // under 1 % of the candidates.  A warp with one to kC1Rows such rows copies their
      // potentials to shared memory and its 32 lanes evaluate them together, one row at a time,
      // after the hand-off (c1 path); more rows take the per-lane path inside the group loop.
      const bool statrow = cond1 || (need23 && valid && nsc2 <= 1);
      const uint32_t smask = __ballot_sync(0xffffffffu, statrow);
      const int nstat = __popc(smask);
      const bool c1path = nstat >= 1 && nstat <= kC1Rows;
      const bool statsB = nstat > kC1Rows;
      const bool vcw_needed = statsB && __any_sync(0xffffffffu, cond1);
      // a statistics row's slot: its rank among the warp's statistics rows (lowest lane first)
      float* c1buf = S.c1row[warp - kWE][0] + 128 * __popc(smask & ((1u << lane) - 1u));
      TRE(1, tl, 1);
      TRE2(tl, 1, 1);
      float linf2 = 0.f, minab2 = 3.0e38f, vcamb = 3.0e38f;
      if (!statsB) {
        // pass B, two groups (32 columns) per step: one 32-column load and store, and two
        // independent split chains for the scheduler to interleave.  Half 1 starts with groups
        // 14-15 (15's columns become the layer-3 accumulator, its h2 goes to the shared-memory
        // tail tiles).
#pragma unroll 1
        for (int ip = 0; ip < 4; ip++) {
          const int g0 = h ? (ip == 0 ? 14 : 6 + 2 * ip) : 2 * ip;
          uint32_t v[32];
#if MLPV_EXP == 106
#pragma unroll
          for (int j = 0; j < 32; j++) v[j] = (uint32_t)(j + ip) * lane;
#else
          tmem_ld32(R2 + loff + 16u * g0, v);
          tmem_ld_wait();
#endif
          if (h && ip == 0) {                              // group 15 has left TMEM: layer 3 may use its columns
            fence_before();
            __syncwarp();
            if (lane == 0) arrive_leader(&S.h2_kb[0], rank);
          }
          if (c1path && statrow) {
            float4* dst = reinterpret_cast<float4*>(c1buf + 16 * (g0 - 8 * h));
#pragma unroll
            for (int k = 0; k < 8; k++)
              dst[k] = make_float4(__uint_as_float(v[4 * k]), __uint_as_float(v[4 * k + 1]), __uint_as_float(v[4 * k + 2]),
                                   __uint_as_float(v[4 * k + 3]));
          }
          uint32_t hl[32];                                   // [hi g0 | lo g0 | hi g0+1 | lo g0+1]
#pragma unroll
          for (int k = 0; k < 8; k++) {
            split_pair(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]), hl[k], hl[8 + k]);
            split_pair(__uint_as_float(v[16 + 2 * k]), __uint_as_float(v[16 + 2 * k + 1]), hl[16 + k], hl[24 + k]);
          }
          if (g0 < 14) {
            if (MLPV_EXP != 106) tmem_st32(R2 + loff + 16u * g0, hl);
            else if (hl[3] == 0x12345u) S.sc2[0][r] = hl[5];
          } else {
            uint32_t h14[16];
#pragma unroll
            for (int k = 0; k < 16; k++) h14[k] = hl[k];
            tmem_st16(R2 + loff + 16u * g0, h14);
            *reinterpret_cast<uint4*>(sT + none16_off(r, 0)) = make_uint4(hl[16], hl[17], hl[18], hl[19]);
            *reinterpret_cast<uint4*>(sT + none16_off(r, 8)) = make_uint4(hl[20], hl[21], hl[22], hl[23]);
            *reinterpret_cast<uint4*>(sT + kBiasTile + none16_off(r, 0)) = make_uint4(hl[24], hl[25], hl[26], hl[27]);
            *reinterpret_cast<uint4*>(sT + kBiasTile + none16_off(r, 8)) = make_uint4(hl[28], hl[29], hl[30], hl[31]);
            fence_proxy_async();
          }
          if (h ? ip >= 2 : (ip & 1)) {                     // K block (g0 + 1) >> 2 complete on this half
            const int kb = h ? ip : ip >> 1;
            tmem_st_wait();
            fence_before();
            __syncwarp();
            if (lane == 0) arrive_leader(&S.h2_kb[kb], rank);
            TRE(1, tl, 2 + kb);
            TRE2(tl, 1, 2 + kb);
          }
        }
      } else {
        // pass B, per group (warps computing the statistics per lane): half 1 starts with group 15
        uint32_t vbuf[2][16];
        const int gfirst = h ? 15 : 0;
        tmem_ld16(R2 + loff + 16u * gfirst, vbuf[0]);
        tmem_ld_wait();
        if (h) {                                           // group 15 has left TMEM: layer 3 may use its columns
          fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(&S.h2_kb[0], rank);
        }
#pragma unroll 2
        for (int i = 0; i < 8; i++) {
          const int g = h ? (i == 0 ? 15 : 7 + i) : i;
          uint32_t (&v)[16] = vbuf[i & 1];
          if (i < 7) {
            const int gn = h ? 8 + i : i + 1;
            tmem_ld16(R2 + loff + 16u * gn, vbuf[(i + 1) & 1]);
          }
          TRP(tl, i, 0);
          if (c1path && statrow) {
            float4* dst = reinterpret_cast<float4*>(c1buf + 16 * (g - 8 * h));
            dst[0] = make_float4(__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]), __uint_as_float(v[3]));
            dst[1] = make_float4(__uint_as_float(v[4]), __uint_as_float(v[5]), __uint_as_float(v[6]), __uint_as_float(v[7]));
            dst[2] = make_float4(__uint_as_float(v[8]), __uint_as_float(v[9]), __uint_as_float(v[10]), __uint_as_float(v[11]));
            dst[3] = make_float4(__uint_as_float(v[12]), __uint_as_float(v[13]), __uint_as_float(v[14]), __uint_as_float(v[15]));
          }
          if (statsB) {
            const float4* ub = reinterpret_cast<const float4*>(S.ub2 + 16 * g);
            float uu[16], d[16];
#pragma unroll
            for (int k = 0; k < 4; k++) {
              const float4 b4 = ub[k];
              const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
              for (int j = 0; j < 4; j++) {
                uu[4 * k + j] = __uint_as_float(v[4 * k + j]);
                d[4 * k + j] = uu[4 * k + j] - bb[j];
              }
            }
            linf2 = max_abs16(linf2, d);
            minab2 = min_abs16(minab2, uu);
            if (vcw_needed) {
              // value change |d| >= tg2 <=> sign bit of the exact difference |d| - tg2 is clear
              float dt[16];
#pragma unroll
              for (int j = 0; j < 16; j++) dt[j] = fabsf(d[j]) - tg2;
              vcamb = min_abs16(vcamb, dt);
              uint32_t lt[16];
#pragma unroll
              for (int j = 0; j < 16; j++) lt[j] = __float_as_uint(dt[j]);
              S.vc2[g][r] = (uint16_t)~sign16(lt);
            }
          }
          TRP(tl, i, 1);
          uint32_t hl[16];                                   // [hi (8 cols) | lo (8 cols)]
#pragma unroll
          for (int k = 0; k < 8; k++) split_pair(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]), hl[k], hl[8 + k]);
          TRP(tl, i, 2);
          if (g < 15) {
            tmem_st16(R2 + loff + 16u * g, hl);
          } else {
            *reinterpret_cast<uint4*>(sT + none16_off(r, 0)) = make_uint4(hl[0], hl[1], hl[2], hl[3]);
            *reinterpret_cast<uint4*>(sT + none16_off(r, 8)) = make_uint4(hl[4], hl[5], hl[6], hl[7]);
            *reinterpret_cast<uint4*>(sT + kBiasTile + none16_off(r, 0)) = make_uint4(hl[8], hl[9], hl[10], hl[11]);
            *reinterpret_cast<uint4*>(sT + kBiasTile + none16_off(r, 8)) = make_uint4(hl[12], hl[13], hl[14], hl[15]);
            fence_proxy_async();
          }
          if (g == 3 || g == 7 || g == 11 || g == 14) {
            tmem_st_wait();
            fence_before();
            __syncwarp();
            if (lane == 0) arrive_leader(&S.h2_kb[g >> 2], rank);
            TRE(1, tl, 2 + (g >> 2));
            TRE2(tl, 1, 2 + (g >> 2));
          }
          TRP(tl, i, 3);
          tmem_ld_wait();
          TRP(tl, i, 4);
        }
      }
      if (et == 0) TR(tl, 11);
      TRE2(tl, 1, 6);
      if (c1path) {
        // one statistics row at a time (slot order = lane order); lane l: neurons 4l..4l+3 of this
        // half, the same fp32 operations as the per-lane path
        __syncwarp();
        uint32_t rest = smask;
#pragma unroll 1
        for (int slot = 0; rest; slot++) {
        const int owner = __ffs(rest) - 1;
        rest &= rest - 1u;
        const float4 u4 = reinterpret_cast<const float4*>(S.c1row[warp - kWE][slot])[lane];
        const float4 b4 = reinterpret_cast<const float4*>(S.ub2 + 128 * h)[lane];
        const float uu[4] = {u4.x, u4.y, u4.z, u4.w}, bb[4] = {b4.x, b4.y, b4.z, b4.w};
        uint32_t nib = 0;
        float mnu = 3.0e38f, mnv = 3.0e38f, mxd = 0.f;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const float d = uu[k] - bb[k];
          const float dt = fabsf(d) - tg2;
          nib |= (__float_as_uint(dt) >> 31 ^ 1u) << k;
          mnu = fminf(mnu, fabsf(uu[k]));
          mnv = fminf(mnv, fabsf(dt));
          mxd = fmaxf(mxd, fabsf(d));
        }
        // |x| >= 0: float order = unsigned order of the bits
        const float rmnu = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(mnu)));
        const float rmnv = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(mnv)));
        const float rmxd = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(mxd)));
        uint32_t w[4];
#pragma unroll
        for (int pp = 0; pp < 4; pp++)
          w[pp] = __reduce_or_sync(0xffffffffu, (lane >> 3) == pp ? nib << (4 * (lane & 7)) : 0u);
        if (lane == owner) {
          minab2 = fminf(minab2, rmnu);
          vcamb = fminf(vcamb, rmnv);
          linf2 = fmaxf(linf2, rmxd);
#pragma unroll
          for (int pp = 0; pp < 4; pp++) {
            S.vc2[8 * h + 2 * pp][r] = (uint16_t)w[pp];
            S.vc2[8 * h + 2 * pp + 1][r] = (uint16_t)(w[pp] >> 16);
          }
        }
        }
      }
      if (slow2) pair_exchange_f(S, h, r, linf2, minab2, vcamb, 9 + q);
      minab2 = fminf(minab2, S.minub2);
      // pair (1, 2): SS / SV row i* (nsc1 == 1) or VS / VV column masks (nsc1 == 0), reading C8;
      // each half updates the words of its own neurons
      if (cond1) {
        const bool certain = !amb1 && minab2 >= tau1 && vcamb >= tau1;
        const uint32_t* off = a.cov.off[a.pair12];
#pragma unroll
        for (int pp = 0; pp < 4; pp++) {
          const int p = 4 * h + pp;
          uint32_t is, iv;
          if (nsc1 == 1) { is = off[0] + istar1 * 8 + p; iv = off[1] + istar1 * 8 + p; }
          else { is = off[2] + p; iv = off[3] + p; }
          const uint32_t scw = S.sc2[p][r];
          if (scw) { atomicOr(&a.res.cov_all[is], scw); if (certain) atomicOr(&a.res.cov_certain[is], scw); }
          const uint32_t vcw = ((uint32_t)S.vc2[2 * p][r] | ((uint32_t)S.vc2[2 * p + 1][r] << 16)) & ~scw;
          if (vcw) { atomicOr(&a.res.cov_all[iv], vcw); if (certain) atomicOr(&a.res.cov_certain[iv], vcw); }
        }
      }
      if (h == 0) continue;                                // E3 is done by half 1
      const bool cond2 = need23 && valid && ((nsc2 == 1) || (nsc2 == 0 && linf2 >= th2));
      const bool amb2 = minab2 < tau1 || (nsc2 == 0 && fabsf(linf2 - th2) < tau1);
      // =========================== E3: logits -> pair (2, 3), argmax, property, counts
      if (et == 128) mbar_wait_sleep(&S.acc3_full, tl & 1u, 64);
      named_bar(5, 128);
      if (et == 128) TR(tl, 12);
      fence_after();
      uint32_t v[16];
      tmem_ld16(R3 + loff, v);
      tmem_ld_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader(&S.acc2_free, rank);
      const int n3 = a.n3;
      float y[16];
#pragma unroll
      for (int i = 0; i < 16; i++) y[i] = __uint_as_float(v[i]) + S.b3[i];
      if (eval) {
        if (valid) {
#pragma unroll
          for (int i = 0; i < 16; i++) if (i < n3) a.eval_out[cidx * a.T + kN1 + kN2 + i] = y[i];
        }
      } else {
        const int bcls = S.bcls;
        if (cond2) {
          uint32_t neg = 0, vcw = 0;
          float minab3 = S.minub3, vcamb3 = 3.0e38f;
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
          const bool certain = !amb2 && minab3 >= tau2 && vcamb3 >= tau2;
          const uint32_t* off = a.cov.off[a.pair23];
          uint32_t is, iv;
          if (nsc2 == 1) { is = off[0] + istar2; iv = off[1] + istar2; }
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
        if (a.prop.kind == MLPV_PROP_THRESHOLD_LITERAL || a.prop.kind == MLPV_PROP_THRESHOLD_LITERAL_ALL) {
          const int D = a.prop.target >= 0 ? a.prop.target : bcls;
          bool any = false, all = true;
          float yD = 0.f;
#pragma unroll
          for (int i = 0; i < 16; i++)
            if (i < n3) {
              if (i == D) yD = y[i];
              if (i != D && y[i] > a.prop.V_f) any = true;
              if (i != D && !(y[i] > a.prop.V_f)) all = false;
              if (fabsf(y[i] - a.prop.V_f) < a.cov.near_tie) flag = true;
            }
          viol = yD < a.prop.V_f && (a.prop.kind == MLPV_PROP_THRESHOLD_LITERAL_ALL ? all : any);
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
      if (et == 128) TR(tl, 13);
    }
  }
  fence_before();
  __syncthreads();
  cluster_sync();
  fence_after();
  if (warp == kWIss) tmem_dealloc2(tb, 512);
}

}  // namespace f3

#ifdef MLPV_TRACE
extern "C" int mlpv_f3_trace_read(void* host) {
  return (int)cudaMemcpyFromSymbol(host, f3::g_trace, sizeof f3::g_trace);
}
extern "C" int mlpv_f3_trace_iss_read(void* host) {
  return (int)cudaMemcpyFromSymbol(host, f3::g_trace_iss, sizeof f3::g_trace_iss);
}
extern "C" int mlpv_f3_trace_epi_read(void* host) {
  return (int)cudaMemcpyFromSymbol(host, f3::g_trace_epi, sizeof f3::g_trace_epi);
}
extern "C" int mlpv_f3_trace_grp_read(void* host) {
  return (int)cudaMemcpyFromSymbol(host, f3::g_trace_grp, sizeof f3::g_trace_grp);
}
extern "C" int mlpv_f3_trace_e2_read(void* host) {
  return (int)cudaMemcpyFromSymbol(host, f3::g_trace_e2, sizeof f3::g_trace_e2);
}
extern "C" int mlpv_f3_trace_done_read(void* host) {
  return (int)cudaMemcpyFromSymbol(host, f3::g_trace_done, sizeof f3::g_trace_done);
}
extern "C" int mlpv_f3_trace_e1p_read(void* host) {
  return (int)cudaMemcpyFromSymbol(host, f3::g_trace_e1p, sizeof f3::g_trace_e1p);
}
extern "C" int mlpv_f3_trace_gen_read(void* host) {
  return (int)cudaMemcpyFromSymbol(host, f3::g_trace_gen, sizeof f3::g_trace_gen);
}
#endif

// ------------------------------------------------------------------------------------------- host
bool fused3_applicable(const DevNet& net) {
  return net.numeric == MLPV_NUM_BF16 && net.L == 3 && net.sizes[1] == f3::kN1 && net.sizes[2] == f3::kN2 &&
         net.sizes[3] <= f3::kN3P && net.sizes[0] % 2 == 0 && net.sizes[0] <= f3::kMaxN0;
}

static size_t sw128_h(uint32_t row, uint32_t byte) {
  return (row >> 3) * 1024u + (row & 7u) * 128u + ((((byte >> 4) ^ row) & 7u) << 4) + (byte & 15u);
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
static float h2f(uint16_t u) {
  __half h;
  memcpy(&h, &u, 2);
  return __half2float(h);
}

// Device weight block of k_fused3 (host-side, once per handle), see f3::Layout:
//   stream [rank][nkb1 + 4][16 KB]: W1 rows [128 rank, +128) per K block (bias hi/mid/lo at K = n0..n0+2),
//          then W2 (fp16) rows [128 rank, +128) per K block of 64 layer-1 neurons;
//   w3 [rank][8][1 KB]: W3 (fp16) rows [8 rank, +8) (rows >= n3 zero), chunk p = [W3[:, 32p..] | same];
//   ones [16 KB]: A operand of the layer-2 bias MMA (1.0 at K = 0, 1 of every row);
//   bias2 [rank][16 KB]: B operand, row n = [RN_f16(b2[n]), RN_f16(b2[n] - hi), 0 ...] (K-major).
cudaError_t prepare_fused3(const DevNet& net, const void* const* W_host, const void* const* b_host, void** blk_dev) {
  const int n0 = net.sizes[0], n3 = net.sizes[3];
  const f3::Layout L = f3::layout_of(n0);
  std::vector<uint8_t> blk(L.total, 0);
  const uint16_t* W1 = static_cast<const uint16_t*>(W_host[0]);
  const uint16_t* W2 = static_cast<const uint16_t*>(W_host[1]);
  const uint16_t* W3 = static_cast<const uint16_t*>(W_host[2]);
  const float* b2 = static_cast<const float*>(b_host[1]);
  auto put16 = [&](uint8_t* tile, int row, int kelem, uint16_t v) {
    const size_t o = sw128_h((uint32_t)row, (uint32_t)(2 * (kelem % 64)));
    tile[o] = (uint8_t)(v & 0xFF);
    tile[o + 1] = (uint8_t)(v >> 8);
  };
  uint8_t* st = blk.data() + L.stream;
  for (int rk = 0; rk < 2; rk++) {
    for (int rr = 0; rr < 128; rr++) {
      const int n = 128 * rk + rr;
      // W1 in fp16 (the A operand holds fp16 levels): exact for |w| >= 2^-17, the smaller weights
      // round with absolute error <= 2^-25 (reading C19); K beyond n0 stays zero
      for (int k = 0; k < n0; k++)
        put16(st + ((size_t)rk * L.nst + k / 64) * f3::kTile, rr, k, f2h(bf2f(W1[(size_t)n * n0 + k])));
      for (int k = 0; k < f3::kN1; k++) {
        const uint16_t h = f2h(bf2f(W2[(size_t)n * f3::kN1 + k]));      // exact for |w| >= 2^-17
        put16(st + ((size_t)rk * L.nst + L.nkb1 + k / 64) * f3::kTile, rr, k, h);
      }
      // bias-2 B operand: row rr of this CTA's half
      const float b = b2[n];
      const uint16_t bh = f2h(b);
      const uint16_t bl = f2h(b - h2f(bh));
      uint8_t* bt = blk.data() + L.bias2 + (size_t)rk * f3::kBiasTile;
      memcpy(bt + tc::none16_off((uint32_t)rr, 0), &bh, 2);
      memcpy(bt + tc::none16_off((uint32_t)rr, 1), &bl, 2);
    }
    for (int rr = 0; rr < 8; rr++) {
      const int n = 8 * rk + rr;
      for (int p = 0; p < f3::kChunks; p++)
        for (int i = 0; i < 32; i++) {
          const uint16_t h = n < n3 ? f2h(bf2f(W3[(size_t)n * f3::kN2 + 32 * p + i])) : (uint16_t)0;
          uint8_t* tile = blk.data() + L.w3 + ((size_t)rk * f3::kChunks + p) * f3::kW3Chunk;
          for (int half = 0; half < 2; half++) {
            const size_t o = sw128_h((uint32_t)rr, (uint32_t)(64 * half + 2 * i));
            tile[o] = (uint8_t)(h & 0xFF);
            tile[o + 1] = (uint8_t)(h >> 8);
          }
        }
    }
  }
  for (int rr = 0; rr < 128; rr++) {
    const uint16_t one = 0x3C00u;                         // fp16 1.0
    memcpy(blk.data() + L.ones + tc::none16_off((uint32_t)rr, 0), &one, 2);
    memcpy(blk.data() + L.ones + tc::none16_off((uint32_t)rr, 1), &one, 2);
  }
  // the setmaxnreg budget assumes this register allocation (checked once per handle)
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, f3::k_fused3);
  if (e != cudaSuccess) return e;
  if (fa.numRegs != f3::kRegLaunch) return cudaErrorInvalidConfiguration;
  e = cudaMalloc(blk_dev, blk.size());
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*blk_dev, blk.data(), blk.size(), cudaMemcpyHostToDevice);
}

cudaError_t launch_fused3(const DevNet& net, const void* blk, const void* bases, int n_base, const DevPert& pert,
                          const DevProp& prop, const DevCov& cov, const DevResult& res, BaseWS ws,
                          const uint64_t* eval_idx, int64_t eval_n, int eval_base, void* eval_out, int num_sms,
                          cudaStream_t st) {
  f3::Args a;
  memset(&a, 0, sizeof a);
  a.n0 = net.sizes[0];
  a.n3 = net.sizes[3];
  a.lay = f3::layout_of(a.n0);
  a.nkb1 = a.lay.nkb1;
  a.nk16 = a.lay.nk16;
  a.wblk = static_cast<const uint8_t*>(blk);
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
  a.clamp = pert.kind == MLPV_PERT_PHILOX_CLAMP ? 1 : 0;
  if (a.clamp) {
    a.stepS = ldexpf(1.0f, -pert.clamp_s);             // the A operand is d * 2^s
    a.cm2 = pert.clamp_m2;
    a.cc2 = pert.clamp_c2;
    a.clampc = ws.clampc;
    const double o15 = pert.origin_d + 15.0 * pert.step_d;
    a.offlo = (float)std::ldexp(std::fmin(pert.origin_d, o15), pert.clamp_s);
    a.offhi = (float)std::ldexp(std::fmax(pert.origin_d, o15), pert.clamp_s);
  } else {
    a.stepS = (float)(pert.step_d * 16777216.0);       // step * 2^24 (the levels are l * 2^-24)
  }
  a.base1 = ws.base1;
  {
    uint32_t k0 = (uint32_t)pert.seed, k1 = (uint32_t)(pert.seed >> 32);
    for (int r = 0; r < 10; r++) {
      a.rk[2 * r] = k0;
      a.rk[2 * r + 1] = k1;
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
  }
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
