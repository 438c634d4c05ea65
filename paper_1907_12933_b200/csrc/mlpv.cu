// mlpv.cu -- host side of the C ABI declared in include/mlpv.h: argument validation, device
// copies of the net, per-call workspace, and the launch sequence of the check
//   init results -> K0 base prologue -> (tau) -> enumeration kernel (k_small / k_large).
// No torch types; plain pointers and sizes only.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "mlpv_internal.cuh"

using namespace mlpv;

namespace mlpv {
// k_large.cu
cudaError_t launch_large(const DevNet& net, const void* const* Wt, void* scratch, const void* bases, int n_base,
                         const DevPert& pert, const DevProp& prop, const DevCov& cov, const DevResult& res,
                         BaseWS ws, const uint64_t* eval_idx, int64_t eval_n, int eval_base, void* eval_out,
                         int num_sms, cudaStream_t st, bool* supported, std::string* why);
cudaError_t prepare_large(const DevNet& net, const void* const* W_host, const void* const* b_host, void** Wt_dev,
                          size_t* scratch_per_cta, std::string* why);
}  // namespace mlpv

struct mlpv_ctx {
  int device = 0;
  int num_sms = 148;
  DevNet net{};
  std::vector<void*> allocs;          // device allocations owned by the handle
  void* Wt[kMaxL] = {};               // tensor-core layouts of the weights (large path)
  bool large_ready = false;
  std::string large_why;
  void* ws = nullptr;
  size_t ws_size = 0;
  mlpv_status sticky = MLPV_OK;
  std::string err;
  std::vector<double> acc_scale;
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;   // mlpv_profile
  uint64_t launches = 0;
  void* steps_dev = nullptr;          // incremental bounds: [kMaxSteps] r2 values (NEXT-2)
  void* scratch = nullptr;            // k_large activation scratch: [num_sms][scratch_per_cta], zeroed once
  uint32_t* dev_status = nullptr;     // device status word (input errors found on the device; mlpv_sync)
};

static thread_local std::string g_err;

static mlpv_status fail(mlpv_ctx* h, mlpv_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) h->err = buf; else g_err = buf;
  return s;
}

static mlpv_status cuda_fail(mlpv_ctx* h, cudaError_t e, const char* what) {
  if (h) h->sticky = MLPV_E_CUDA;
  return fail(h, MLPV_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CUDA_TRY(h, call, what)                      \
  do {                                               \
    cudaError_t e_ = (call);                         \
    if (e_ != cudaSuccess) return cuda_fail(h, e_, what); \
  } while (0)

static size_t in_elem(int numeric) {
  return numeric == MLPV_NUM_FP32 ? 4 : (numeric == MLPV_NUM_INT8 ? 1 : 2);
}
static size_t w_elem(int numeric) {
  return numeric == MLPV_NUM_FP32 ? 4 : (numeric == MLPV_NUM_INT8 ? 1 : 2);
}
static bool is_fixed(int numeric) { return numeric == MLPV_NUM_Q4_12 || numeric == MLPV_NUM_INT8; }

static double bf16_to_double(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static bool f16_exact(double v, uint16_t* bits) {     // v is an fp16 value (RN round trip)
  const float f = (float)v;
  if ((double)f != v) return false;
  const __half hh = __float2half_rn(f);
  if ((double)__half2float(hh) != v) return false;
  memcpy(bits, &hh, 2);
  return true;
}
static bool is_philox(int kind) {
  return kind == MLPV_PERT_PHILOX_LATTICE || kind == MLPV_PERT_PHILOX_BOX || kind == MLPV_PERT_PHILOX_CLAMP;
}
static bool is_bf16_value(double v) {
  float f = (float)v;
  if ((double)f != v) return false;
  uint32_t u;
  memcpy(&u, &f, 4);
  return (u & 0xFFFFu) == 0;
}

// ---------------------------------------------------------------------------------------- create
extern "C" mlpv_status mlpv_create(const mlpv_net* net, const mlpv_quant* quant, int device, mlpv_t* out) {
  if (!out) return fail(nullptr, MLPV_E_INVALID, "out is NULL");
  *out = nullptr;
  if (!net || !quant) return fail(nullptr, MLPV_E_INVALID, "net or quant is NULL");
  const int L = net->n_layers;
  if (L < 1 || L > MLPV_MAX_LAYERS) return fail(nullptr, MLPV_E_INVALID, "net.n_layers = %d (1..%d)", L, MLPV_MAX_LAYERS);
  if (!net->sizes || !net->W || !net->b) return fail(nullptr, MLPV_E_INVALID, "net.sizes / net.W / net.b is NULL");
  for (int l = 0; l <= L; l++)
    if (net->sizes[l] < 1 || net->sizes[l] > (1 << 20)) return fail(nullptr, MLPV_E_SHAPE, "net.sizes[%d] = %d", l, net->sizes[l]);
  if (net->sizes[L] > MLPV_MAX_CLASSES) return fail(nullptr, MLPV_E_SHAPE, "net.sizes[%d] = %d classes (max %d)", L, net->sizes[L], MLPV_MAX_CLASSES);
  const int num = quant->numeric;
  if (num < 0 || num > 3) return fail(nullptr, MLPV_E_INVALID, "quant.numeric = %d", num);
  const int act = net->hidden_act;
  if (act < 0 || act > 2) return fail(nullptr, MLPV_E_INVALID, "net.hidden_act = %d", act);
  const bool act_ok = (num == MLPV_NUM_FP32 && (act == MLPV_ACT_SIGMOID || act == MLPV_ACT_RELU)) ||
                      (num == MLPV_NUM_BF16 && act == MLPV_ACT_RELU) ||
                      (num == MLPV_NUM_Q4_12 && (act == MLPV_ACT_PL_SIGMOID || act == MLPV_ACT_RELU)) ||
                      (num == MLPV_NUM_INT8 && act == MLPV_ACT_RELU);
  if (!act_ok) return fail(nullptr, MLPV_E_UNSUPPORTED, "numeric %d with hidden activation %d is not built", num, act);
  if (act == MLPV_ACT_PL_SIGMOID && !quant->sigmoid_knots) return fail(nullptr, MLPV_E_INVALID, "quant.sigmoid_knots is NULL");
  if (num == MLPV_NUM_INT8 && L > 1 && !quant->requant_shift) return fail(nullptr, MLPV_E_INVALID, "quant.requant_shift is NULL");
  if (num == MLPV_NUM_INT8 && !quant->acc_scale) return fail(nullptr, MLPV_E_INVALID, "quant.acc_scale is NULL (required for INT8)");
  if (num == MLPV_NUM_INT8)
    for (int l = 0; l + 1 < L; l++)
      if (quant->requant_shift[l] < 0 || quant->requant_shift[l] > 24) return fail(nullptr, MLPV_E_INVALID, "quant.requant_shift[%d] = %d", l, quant->requant_shift[l]);
  for (int l = 0; l < L; l++) {
    if (!net->W[l] || !net->b[l]) return fail(nullptr, MLPV_E_INVALID, "net.W[%d] or net.b[%d] is NULL", l, l);
    if (quant->acc_scale && !(quant->acc_scale[l] > 0.0 && std::isfinite(quant->acc_scale[l])))
      return fail(nullptr, MLPV_E_INVALID, "quant.acc_scale[%d] = %g", l, quant->acc_scale[l]);
  }
  if (act == MLPV_ACT_PL_SIGMOID)
    for (int m = 0; m + 1 < 129; m++)
      if (quant->sigmoid_knots[m] > quant->sigmoid_knots[m + 1] || quant->sigmoid_knots[m] < 0)
        return fail(nullptr, MLPV_E_INVALID, "quant.sigmoid_knots not monotone / negative at %d", m);
  // finiteness (float) and the fixed-point accumulator bound (reading C16/C18):
  // sum_j |w_ij| * x_max + |b_i| < 2^30 for every neuron, so every potential and every
  // base-vs-candidate difference fits in int32.
  double hbound = 1.0;                       // BF16: bound on |input| of layer l (images in [0, 1])
  for (int l = 0; l < L; l++) {
    const int nl = net->sizes[l + 1], fan = net->sizes[l];
    double nbound = 0.0;
    double xmax;
    // Q4.12 images are normalised: raw inputs in [0, 4096]
    if (num == MLPV_NUM_Q4_12) xmax = l == 0 ? 4096.0 : (act == MLPV_ACT_PL_SIGMOID ? 4096.0 : 32767.0);
    else xmax = 255.0;
    for (int i = 0; i < nl; i++) {
      double s = 0.0;
      for (int j = 0; j < fan; j++) {
        const size_t e = (size_t)i * fan + j;
        double w;
        switch (num) {
          case MLPV_NUM_FP32: w = static_cast<const float*>(net->W[l])[e]; break;
          case MLPV_NUM_BF16: w = bf16_to_double(static_cast<const uint16_t*>(net->W[l])[e]); break;
          case MLPV_NUM_Q4_12: w = static_cast<const int16_t*>(net->W[l])[e]; break;
          default: w = static_cast<const int8_t*>(net->W[l])[e]; break;
        }
        if (!std::isfinite(w)) return fail(nullptr, MLPV_E_INVALID, "net.W[%d][%d][%d] is not finite", l, i, j);
        s += std::fabs(w);
      }
      if (num == MLPV_NUM_BF16 && l + 1 < L) {
        // hidden activations (and their base differences) travel as fp16 hi + lo into the next
        // tensor-core layer: the worst case sum |w| x_max + |b| must stay below the fp16 range
        // (inputs in [0, 1]; later layers bounded by this layer's bound, below)
        const double bb = std::fabs((double)static_cast<const float*>(net->b[l])[i]);
        if (s * hbound + bb >= 32768.0)
          return fail(nullptr, MLPV_E_UNSUPPORTED, "BF16 layer %d neuron %d: worst-case |potential| %.0f exceeds the fp16 "
                      "carrier range of the tensor-core path", l + 1, i, s * hbound + bb);
        nbound = std::max(nbound, s * hbound + bb);
      }
      if (is_fixed(num)) {
        const double bb = std::fabs((double)static_cast<const int32_t*>(net->b[l])[i]);
        if (s * xmax + bb >= 1073741824.0)
          return fail(nullptr, MLPV_E_OVERFLOW, "layer %d neuron %d: worst-case |accumulator| %.0f >= 2^30", l + 1, i, s * xmax + bb);
      } else if (!std::isfinite(static_cast<const float*>(net->b[l])[i])) {
        return fail(nullptr, MLPV_E_INVALID, "net.b[%d][%d] is not finite", l, i);
      }
    }
    hbound = nbound;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(nullptr, MLPV_E_CUDA, "no CUDA device");
  if (device < 0 || device >= ndev) return fail(nullptr, MLPV_E_INVALID, "device %d (have %d)", device, ndev);
  mlpv_ctx* h = new mlpv_ctx();
  h->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { delete h; return fail(nullptr, MLPV_E_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e)); }
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  DevNet& d = h->net;
  d.L = L; d.numeric = num; d.act = act;
  int off = 0;
  for (int l = 0; l <= L; l++) d.sizes[l] = net->sizes[l];
  for (int l = 1; l <= L; l++) { d.loff[l] = off; off += net->sizes[l]; }
  d.trace_len = off;
  auto dev_copy = [&](const void* src, size_t bytes, void** dst) -> bool {
    if (cudaMalloc(dst, bytes) != cudaSuccess) return false;
    h->allocs.push_back(*dst);
    return cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
  };
  for (int l = 0; l < L; l++) {
    void* p;
    if (!dev_copy(net->W[l], w_elem(num) * (size_t)net->sizes[l + 1] * net->sizes[l], &p)) { mlpv_destroy(h); return fail(nullptr, MLPV_E_OOM, "device copy of W[%d]", l); }
    d.W[l] = p;
    if (!dev_copy(net->b[l], 4 * (size_t)net->sizes[l + 1], &p)) { mlpv_destroy(h); return fail(nullptr, MLPV_E_OOM, "device copy of b[%d]", l); }
    d.b[l] = p;
    d.shift[l] = (num == MLPV_NUM_INT8 && l + 1 < L) ? quant->requant_shift[l] : 0;
  }
  d.knots = nullptr;
  if (act == MLPV_ACT_PL_SIGMOID) {
    void* p;
    if (!dev_copy(quant->sigmoid_knots, 129 * 2, &p)) { mlpv_destroy(h); return fail(nullptr, MLPV_E_OOM, "device copy of knots"); }
    d.knots = static_cast<const int16_t*>(p);
  }
  h->acc_scale.resize(L);
  for (int l = 0; l < L; l++)
    h->acc_scale[l] = quant->acc_scale ? quant->acc_scale[l] : (num == MLPV_NUM_Q4_12 ? 1.0 / 16777216.0 : 1.0);
  // tensor-core layouts for the large-net path (PHILOX spaces, BF16 / INT8)
  if (num == MLPV_NUM_BF16 || num == MLPV_NUM_INT8) {
    size_t per_cta = 0;
    cudaError_t pe = prepare_large(d, net->W, net->b, h->Wt, &per_cta, &h->large_why);
    if (pe != cudaSuccess) { mlpv_destroy(h); return fail(nullptr, MLPV_E_CUDA, "prepare_large: %s", cudaGetErrorString(pe)); }
    h->large_ready = h->large_why.empty();
    for (int l = 0; l < kMaxL; l++) if (h->Wt[l]) h->allocs.push_back(h->Wt[l]);
    if (h->large_ready && per_cta > 0) {
      // the handle's own activation scratch (K padding zeroed once; the kernels never write it)
      const size_t bytes = per_cta * (size_t)h->num_sms;
      if (cudaMalloc(&h->scratch, bytes) != cudaSuccess) { h->scratch = nullptr; mlpv_destroy(h); return fail(nullptr, MLPV_E_OOM, "k_large scratch of %zu bytes", bytes); }
      h->allocs.push_back(h->scratch);
      if (cudaMemset(h->scratch, 0, bytes) != cudaSuccess) { mlpv_destroy(h); return fail(nullptr, MLPV_E_CUDA, "scratch memset"); }
    }
  }
  {
    void* p = nullptr;
    if (cudaMalloc(&p, 8 * kMaxSteps) != cudaSuccess) { mlpv_destroy(h); return fail(nullptr, MLPV_E_OOM, "steps buffer"); }
    h->allocs.push_back(p);
    h->steps_dev = p;
    if (cudaMalloc(&p, 256) != cudaSuccess) { mlpv_destroy(h); return fail(nullptr, MLPV_E_OOM, "status word"); }
    h->allocs.push_back(p);
    h->dev_status = static_cast<uint32_t*>(p);
    if (cudaMemset(p, 0, 256) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) { mlpv_destroy(h); return fail(nullptr, MLPV_E_CUDA, "status memset"); }
  }
  *out = h;
  return MLPV_OK;
}

extern "C" void mlpv_destroy(mlpv_t h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  for (void* p : h->allocs) cudaFree(p);
  if (h->ws) cudaFree(h->ws);                     // stream-ordered allocation; the device is idle
  delete h;
}

extern "C" const char* mlpv_last_error(mlpv_t h) { return h ? h->err.c_str() : g_err.c_str(); }

extern "C" const char* mlpv_version(void) { return "mlpv 0.1 (sm_100a)"; }

// ---------------------------------------------------------------------------------------- helpers
static mlpv_status build_cov(mlpv_ctx* h, const mlpv_coverage_spec* cov, DevCov* dc) {
  memset(dc, 0, sizeof *dc);
  if (!cov) return fail(h, MLPV_E_INVALID, "coverage spec is NULL");
  const DevNet& n = h->net;
  if (cov->n_pairs < 0 || cov->n_pairs > n.L - 1) return fail(h, MLPV_E_INVALID, "cov.n_pairs = %d (0..%d)", cov->n_pairs, n.L - 1);
  if (cov->n_pairs > 0 && !cov->lower_layer) return fail(h, MLPV_E_INVALID, "cov.lower_layer is NULL");
  if (!(cov->d_value >= 0) || !(cov->d_distance >= 0) || !std::isfinite(cov->d_value) || !std::isfinite(cov->d_distance))
    return fail(h, MLPV_E_INVALID, "cov.d_value / d_distance must be finite and >= 0");
  if (!(cov->near_tie >= 0) || !std::isfinite(cov->near_tie)) return fail(h, MLPV_E_INVALID, "cov.near_tie = %g", cov->near_tie);
  dc->n_pairs = cov->n_pairs;
  uint32_t w = 0;
  for (int p = 0; p < cov->n_pairs; p++) {
    const int k = cov->lower_layer[p];
    if (k < 1 || k >= n.L) return fail(h, MLPV_E_INVALID, "cov.lower_layer[%d] = %d (1..%d)", p, k, n.L - 1);
    for (int q = 0; q < p; q++) if (cov->lower_layer[q] == k) return fail(h, MLPV_E_INVALID, "cov.lower_layer[%d] duplicates pair %d", p, k);
    dc->lower[p] = k;
    const uint32_t wpr = (n.sizes[k + 1] + 31) / 32;
    dc->off[p][0] = w;
    dc->off[p][1] = w + n.sizes[k] * wpr;
    dc->off[p][2] = w + 2 * n.sizes[k] * wpr;
    dc->off[p][3] = w + 2 * n.sizes[k] * wpr + wpr;
    w += 2 * n.sizes[k] * wpr + 2 * wpr;
  }
  dc->n_words = w;
  const bool fx = is_fixed(n.numeric);
  for (int l = 0; l < n.L; l++) {
    // thresholds in potential units (accumulator units for fixed point, RNE)
    dc->tg_f[l] = (float)cov->d_value;
    dc->th_f[l] = (float)cov->d_distance;
    if (fx) {
      const double tg = std::nearbyint(cov->d_value / h->acc_scale[l]);
      const double th = std::nearbyint(cov->d_distance / h->acc_scale[l]);
      if (tg > 2147483647.0 || th > 2147483647.0) return fail(h, MLPV_E_OVERFLOW, "threshold of layer %d exceeds int32 in accumulator units", l + 1);
      dc->tg_i[l] = (int64_t)tg;
      dc->th_i[l] = (int64_t)th;
    }
    dc->tau[l] = cov->tau ? (float)cov->tau[l] : -1.0f;     // < 0: computed on the device
    if (cov->tau && !(cov->tau[l] >= 0)) return fail(h, MLPV_E_INVALID, "cov.tau[%d] = %g", l, cov->tau[l]);
  }
  dc->near_tie = (float)cov->near_tie;
  return MLPV_OK;
}

static uint64_t space_of(const DevNet& n, const mlpv_pert* p) {
  if (p->kind == MLPV_PERT_TUPLE_REPLACE) {
    const uint64_t q = (uint64_t)p->n_levels, n0 = (uint64_t)n.sizes[0];
    return p->tuple == 1 ? n0 * q : n0 * (n0 - 1) / 2 * q * q;
  }
  if (p->kind == MLPV_PERT_SUBSET_OFFSET || p->kind == MLPV_PERT_SUBSET_REPLACE) {
    uint64_t s = 1;
    for (int k = 0; k < p->n_pixels; k++) {
      if (s > (~0ull) / (uint64_t)p->n_levels) return ~0ull;
      s *= (uint64_t)p->n_levels;
    }
    return s;
  }
  return p->n_samples;
}

static mlpv_status build_pert(mlpv_ctx* h, const mlpv_pert* p, DevPert* dp, bool check_range) {
  memset(dp, 0, sizeof *dp);
  if (!p) return fail(h, MLPV_E_INVALID, "perturbation spec is NULL");
  const DevNet& n = h->net;
  const int num = n.numeric;
  dp->kind = p->kind;
  switch (p->kind) {
    case MLPV_PERT_TUPLE_REPLACE:
      if (p->tuple != 1 && p->tuple != 2) return fail(h, MLPV_E_INVALID, "pert.tuple = %d (1 or 2)", p->tuple);
      if (p->tuple == 2 && n.sizes[0] < 2) return fail(h, MLPV_E_SHAPE, "pert.tuple = 2 needs n_0 >= 2");
      // the kernels rank pixel pairs in 32 bits
      if (p->tuple == 2 && (uint64_t)n.sizes[0] * (uint64_t)(n.sizes[0] - 1) / 2 >= (1ull << 32))
        return fail(h, MLPV_E_UNSUPPORTED, "pert.tuple = 2 with n_0 = %d: more than 2^32 pixel pairs", n.sizes[0]);
      if (num == MLPV_NUM_BF16) return fail(h, MLPV_E_UNSUPPORTED, "TUPLE_REPLACE with BF16 is not built (use PHILOX_LATTICE)");
      break;
    case MLPV_PERT_SUBSET_OFFSET:
      if (!is_fixed(num)) return fail(h, MLPV_E_UNSUPPORTED, "SUBSET_OFFSET needs a fixed-point numeric");
      /* fallthrough */
    case MLPV_PERT_SUBSET_REPLACE:
      if (num == MLPV_NUM_BF16) return fail(h, MLPV_E_UNSUPPORTED, "SUBSET spaces with BF16 are not built (use PHILOX_LATTICE)");
      if (p->n_pixels < 1 || p->n_pixels > 16) return fail(h, MLPV_E_INVALID, "pert.n_pixels = %d (1..16)", p->n_pixels);
      if (!p->pixels) return fail(h, MLPV_E_INVALID, "pert.pixels is NULL");
      for (int k = 0; k < p->n_pixels; k++) {
        if (p->pixels[k] < 0 || p->pixels[k] >= n.sizes[0]) return fail(h, MLPV_E_INVALID, "pert.pixels[%d] = %d (n_0 = %d)", k, p->pixels[k], n.sizes[0]);
        if (k > 0 && p->pixels[k] <= p->pixels[k - 1]) return fail(h, MLPV_E_INVALID, "pert.pixels not strictly ascending at %d", k);
      }
      break;
    case MLPV_PERT_PHILOX_LATTICE:
      if (num != MLPV_NUM_BF16 && num != MLPV_NUM_INT8) return fail(h, MLPV_E_UNSUPPORTED, "PHILOX_LATTICE needs BF16 or INT8");
      if (p->n_samples < 1 || p->n_samples > (1ull << 32)) return fail(h, MLPV_E_INVALID, "pert.n_samples = %llu (1..2^32)", (unsigned long long)p->n_samples);
      if (num == MLPV_NUM_BF16) {
        if (!is_bf16_value(p->lattice_step) || !is_bf16_value(p->lattice_origin) || !std::isfinite(p->lattice_step))
          return fail(h, MLPV_E_INVALID, "pert.lattice_step / lattice_origin must be bf16 values");
        dp->step_f = (float)p->lattice_step;
        dp->origin_f = (float)p->lattice_origin;
      } else {
        if (p->lattice_step != std::floor(p->lattice_step) || p->lattice_origin != std::floor(p->lattice_origin) ||
            std::fabs(p->lattice_step) > 255 || std::fabs(p->lattice_origin) > 255)
          return fail(h, MLPV_E_INVALID, "pert.lattice_step / lattice_origin must be integers in [-255, 255]");
        dp->step_i = (int)p->lattice_step;
        dp->origin_i = (int)p->lattice_origin;
      }
      dp->seed = p->seed;
      break;
    case MLPV_PERT_PHILOX_BOX:
      if (num != MLPV_NUM_BF16) return fail(h, MLPV_E_UNSUPPORTED, "PHILOX_BOX is built for BF16 nets");
      if (p->n_samples < 1 || p->n_samples > (1ull << 32)) return fail(h, MLPV_E_INVALID, "pert.n_samples = %llu (1..2^32)", (unsigned long long)p->n_samples);
      if (!std::isfinite(p->lattice_step) || !std::isfinite(p->lattice_origin) || std::fabs(p->lattice_step) > 1.0 ||
          std::fabs(p->lattice_origin) > 1.0)
        return fail(h, MLPV_E_INVALID, "pert.lattice_step / lattice_origin must be finite, |.| <= 1");
      dp->step_f = (float)p->lattice_step;
      dp->origin_f = (float)p->lattice_origin;
      dp->step_d = p->lattice_step;
      dp->origin_d = p->lattice_origin;
      dp->seed = p->seed;
      break;
    case MLPV_PERT_PHILOX_CLAMP: {
      if (num != MLPV_NUM_BF16) return fail(h, MLPV_E_UNSUPPORTED, "PHILOX_CLAMP is built for BF16 nets");
      if (p->n_samples < 1 || p->n_samples > (1ull << 32)) return fail(h, MLPV_E_INVALID, "pert.n_samples = %llu (1..2^32)", (unsigned long long)p->n_samples);
      if (!std::isfinite(p->lattice_step) || !std::isfinite(p->lattice_origin) || std::fabs(p->lattice_step) > 1.0 ||
          std::fabs(p->lattice_origin) > 1.0 || std::fabs(p->lattice_origin + 15.0 * p->lattice_step) > 1.0)
        return fail(h, MLPV_E_INVALID, "pert.lattice_step / lattice_origin must be finite with |origin|, |origin + 15 step| <= 1");
      // the scale s of the fp16 contraction (reading C19): the largest s with
      // step 2^(24+s) <= 65504 and step 2^(24+s), origin 2^s and every offset (origin + l step) 2^s
      // exact in fp16
      bool found = false;
      for (int sc = 24; sc >= -40 && !found; sc--) {
        uint16_t mb, cb, ob;
        const double m = std::ldexp(p->lattice_step, 24 + sc);
        if (std::fabs(m) > 65504.0 || !f16_exact(m, &mb) || !f16_exact(std::ldexp(p->lattice_origin, sc), &cb)) continue;
        bool ok = true;
        for (int l = 0; l < 16 && ok; l++) ok = f16_exact(std::ldexp(p->lattice_origin + l * p->lattice_step, sc), &ob);
        if (!ok) continue;
        dp->clamp_s = sc;
        dp->clamp_m2 = (uint32_t)mb | ((uint32_t)mb << 16);
        dp->clamp_c2 = (uint32_t)cb | ((uint32_t)cb << 16);
        found = true;
      }
      if (!found) return fail(h, MLPV_E_UNSUPPORTED, "PHILOX_CLAMP: the offsets origin + l * step are not exactly representable in fp16 at any scale 2^s");
      dp->step_f = (float)p->lattice_step;
      dp->origin_f = (float)p->lattice_origin;
      dp->step_d = p->lattice_step;
      dp->origin_d = p->lattice_origin;
      dp->seed = p->seed;
      break;
    }
    default:
      return fail(h, MLPV_E_INVALID, "pert.kind = %d", (int)p->kind);
  }
  if (!std::isfinite(p->restrict_l2) || p->restrict_l2 < 0)
    return fail(h, MLPV_E_INVALID, "pert.restrict_l2 = %g (finite, >= 0)", p->restrict_l2);
  if (p->restrict_l2 > 0) {
    // subset / tuple spaces: filtered inside k_small; Philox spaces: a mask pass (k_restrict_mask)
    dp->restrict_on = 1;
    const double b = p->restrict_l2;
    if (is_fixed(num)) {
      const double S = num == MLPV_NUM_Q4_12 ? 4096.0 : 255.0;
      dp->r2_raw = (long long)std::floor(b * b * S * S);
    } else {
      dp->r2_f = b * b;
    }
  }
  if (!is_philox(p->kind)) {
    if (p->n_levels < 1 || p->n_levels > 256) return fail(h, MLPV_E_INVALID, "pert.n_levels = %d (1..256)", p->n_levels);
    if (!p->levels) return fail(h, MLPV_E_INVALID, "pert.levels is NULL");
    for (int q = 0; q < p->n_levels; q++) {
      if (num == MLPV_NUM_FP32) {
        const float v = static_cast<const float*>(p->levels)[q];
        if (!std::isfinite(v)) return fail(h, MLPV_E_INVALID, "pert.levels[%d] is not finite", q);
      } else if (p->kind != MLPV_PERT_SUBSET_OFFSET) {
        const int v = static_cast<const int16_t*>(p->levels)[q];
        // replacement values lie in the input domain: Q4.12 images are normalised (PAPER.md:412,
        // reading C16: raw [0, 4096]; the create-time accumulator bound assumes it), u8 [0, 255]
        const int hi = num == MLPV_NUM_Q4_12 ? 4096 : 255, lo = 0;
        if (v < lo || v > hi) return fail(h, MLPV_E_INVALID, "pert.levels[%d] = %d outside the input range", q, v);
      }
    }
    dp->n_levels = p->n_levels;
  } else {
    dp->n_levels = 16;
  }
  dp->tuple = p->tuple;
  dp->n_pixels = p->n_pixels;
  dp->q2 = (uint64_t)dp->n_levels * dp->n_levels;
  const uint64_t space = space_of(n, p);
  if (space == ~0ull && !is_philox(p->kind)) return fail(h, MLPV_E_INVALID, "perturbation space exceeds 2^64");
  if (check_range) {
    if (p->index_begin > p->index_end || p->index_end > space)
      return fail(h, MLPV_E_INVALID, "pert index range [%llu, %llu) not within [0, %llu)", (unsigned long long)p->index_begin,
                  (unsigned long long)p->index_end, (unsigned long long)space);
  }
  dp->begin = p->index_begin;
  dp->end = p->index_end;
  return MLPV_OK;
}

static mlpv_status build_prop(mlpv_ctx* h, const mlpv_property* pr, DevProp* d) {
  memset(d, 0, sizeof *d);
  if (!pr) return fail(h, MLPV_E_INVALID, "property is NULL");
  const int nL = h->net.sizes[h->net.L];
  if (pr->kind < 0 || pr->kind > 3) return fail(h, MLPV_E_INVALID, "prop.kind = %d", (int)pr->kind);
  if (pr->kind == MLPV_PROP_TARGET_NEVER && (pr->target < 0 || pr->target >= nL)) return fail(h, MLPV_E_INVALID, "prop.target = %d (n_L = %d)", pr->target, nL);
  if ((pr->kind == MLPV_PROP_THRESHOLD_LITERAL || pr->kind == MLPV_PROP_THRESHOLD_LITERAL_ALL) && pr->target >= nL) return fail(h, MLPV_E_INVALID, "prop.target = %d (n_L = %d)", pr->target, nL);
  if (!std::isfinite(pr->V)) return fail(h, MLPV_E_INVALID, "prop.V is not finite");
  d->kind = pr->kind;
  d->target = pr->target;
  d->V_f = (float)pr->V;
  if (is_fixed(h->net.numeric)) {
    const double v = std::nearbyint(pr->V / h->acc_scale[h->net.L - 1]);
    if (std::fabs(v) > 2147483647.0) return fail(h, MLPV_E_OVERFLOW, "prop.V exceeds int32 in accumulator units");
    d->V_i = (int64_t)v;
  }
  return MLPV_OK;
}

// device workspace: [trace n_base*T*4][cls n_base*4][tau 8*4][delta][pixels][levels][base1][clampc].
// Grown with stream-ordered allocation on the caller's stream (no device synchronisation); the
// work of one handle is ordered on one stream at a time (mlpv.h conventions).
static mlpv_status ensure_ws(mlpv_ctx* h, size_t bytes, cudaStream_t st) {
  if (h->ws_size >= bytes) return MLPV_OK;
  if (h->ws) {
    cudaError_t e = cudaFreeAsync(h->ws, st);
    h->ws = nullptr;
    h->ws_size = 0;
    if (e != cudaSuccess) return cuda_fail(h, e, "workspace free");
  }
  size_t want = bytes + bytes / 4 + 4096;
  cudaError_t e = cudaMallocAsync(&h->ws, want, st);
  if (e != cudaSuccess) { h->ws = nullptr; return fail(h, MLPV_E_OOM, "workspace of %zu bytes: %s", want, cudaGetErrorString(e)); }
  h->ws_size = want;
  return MLPV_OK;
}

struct Plan {
  BaseWS ws;
  float* tau_dev;
  int32_t* pixels_dev;
  void* levels_dev;
};

static mlpv_status prepare(mlpv_ctx* h, const void* bases, int n_base, const mlpv_pert* pert, const DevPert& dp,
                           DevCov* dc, Plan* plan, cudaStream_t st, bool need_tau) {
  const DevNet& n = h->net;
  const int T = n.trace_len;
  const bool subset = !is_philox(pert->kind);
  const bool clamp = pert->kind == MLPV_PERT_PHILOX_CLAMP;
  const bool box = pert->kind == MLPV_PERT_PHILOX_BOX || clamp;   // base1 = W1 x + b1 (+ origin W1 1)
  const int S = pert->kind == MLPV_PERT_TUPLE_REPLACE ? n.sizes[0] : pert->n_pixels;
  const size_t delta_bytes = subset ? 4ull * n_base * S * dp.n_levels * n.sizes[1] : 0;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t o_trace = 0, o_cls = al(4ull * n_base * T), o_tau = o_cls + al(4ull * n_base);
  const size_t o_delta = o_tau + al(4 * kMaxL), o_pix = o_delta + al(delta_bytes);
  const size_t o_lv = o_pix + al(4 * 64), o_b1 = o_lv + al(4 * 256);
  const size_t o_cc = o_b1 + (box ? al(4ull * n_base * n.sizes[1]) : 0);
  const size_t total = o_cc + (clamp ? al(32ull * n_base * ((n.sizes[0] + 7) / 8)) : 0);
  mlpv_status s = ensure_ws(h, total, st);
  if (s != MLPV_OK) return s;
  char* w = static_cast<char*>(h->ws);
  plan->ws.trace = w + o_trace;
  plan->ws.cls = reinterpret_cast<int32_t*>(w + o_cls);
  plan->ws.delta = subset ? w + o_delta : nullptr;
  plan->ws.S = S;
  plan->ws.base1 = box ? reinterpret_cast<float*>(w + o_b1) : nullptr;
  plan->ws.clampc = clamp ? reinterpret_cast<uint4*>(w + o_cc) : nullptr;
  plan->ws.status = h->dev_status;
  plan->tau_dev = reinterpret_cast<float*>(w + o_tau);
  plan->pixels_dev = reinterpret_cast<int32_t*>(w + o_pix);
  plan->levels_dev = w + o_lv;
  if (subset) {
    const size_t lv_bytes = (n.numeric == MLPV_NUM_FP32 ? 4 : 2) * (size_t)pert->n_levels;
    // small parameter arrays; synchronous copies (pageable host memory)
    if (pert->kind != MLPV_PERT_TUPLE_REPLACE)
      CUDA_TRY(h, cudaMemcpyAsync(plan->pixels_dev, pert->pixels, 4 * (size_t)pert->n_pixels, cudaMemcpyHostToDevice, st), "copy pixels");
    CUDA_TRY(h, cudaMemcpyAsync(plan->levels_dev, pert->levels, lv_bytes, cudaMemcpyHostToDevice, st), "copy levels");
  }
  DevPert dp2 = dp;
  dp2.pixels = plan->pixels_dev;
  CUDA_TRY(h, launch_base_prologue(n, bases, n_base, dp2, plan->levels_dev, plan->ws, st), "base prologue");
  h->launches++;
  if (need_tau) {
    bool any = false;
    for (int l = 0; l < n.L; l++) any |= dc->tau[l] < 0;
    if (any) {
      CUDA_TRY(h, launch_tau(n, plan->ws.trace, n_base, plan->tau_dev, st), "tau");
      h->launches += 2;                           // k_tau_max + k_tau_final
    }
  }
  return MLPV_OK;
}

static mlpv_status run_kernel(mlpv_ctx* h, const void* bases, int n_base, const mlpv_pert* pert, DevPert dp,
                              const DevProp& dprop, const DevCov& dc, const DevResult& dr, const Plan& plan,
                              const uint64_t* eval_idx, int64_t eval_n, int eval_base, void* eval_out, cudaStream_t st) {
  dp.pixels = plan.pixels_dev;
  bool supported = false;
  cudaError_t e;
  if (h->ev_begin) CUDA_TRY(h, cudaEventRecord(h->ev_begin, st), "profile event");
  if (is_philox(pert->kind)) {
    if (!h->large_ready) return fail(h, MLPV_E_UNSUPPORTED, "large-net path unavailable for this net: %s", h->large_why.c_str());
    std::string why;
    e = launch_large(h->net, h->Wt, h->scratch, bases, n_base, dp, dprop, dc, dr, plan.ws, eval_idx, eval_n, eval_base,
                     eval_out, h->num_sms, st, &supported, &why);
    if (!supported) return fail(h, MLPV_E_UNSUPPORTED, "large-net kernel: %s", why.c_str());
  } else {
    dp.levels = plan.levels_dev;
    supported = false;
    e = cudaSuccess;
    if (!eval_idx && !getenv("MLPV_NO_TC3"))            // small int8 nets: tcgen05 per layer (k_tc3)
      e = launch_tc3(h->net, bases, n_base, dp, dprop, dc, dr, plan.ws, h->num_sms, st, &supported);
    if (!supported && !eval_idx && !getenv("MLPV_NO_WARP3"))   // ... else one warp per candidate (k_warp)
      e = launch_warp3(h->net, n_base, dp, dprop, dc, dr, plan.ws, h->num_sms, st, &supported);
    if (!supported)
      e = launch_small(h->net, bases, n_base, dp, dprop, dc, dr, plan.ws, eval_idx, eval_n, eval_base, eval_out,
                       h->num_sms, st, &supported);
    if (!supported) return fail(h, MLPV_E_UNSUPPORTED, "no small-net kernel for this shape / numeric (L=%d, widths %d,%d,%d)",
                                h->net.L, h->net.sizes[1], h->net.L > 1 ? h->net.sizes[2] : 0, h->net.L > 2 ? h->net.sizes[3] : 0);
  }
  if (e != cudaSuccess) return cuda_fail(h, e, "enumeration kernel");
  h->launches++;
  if (h->ev_end) CUDA_TRY(h, cudaEventRecord(h->ev_end, st), "profile event");
  return MLPV_OK;
}

extern "C" mlpv_status mlpv_profile(mlpv_t h, void* ev_begin, void* ev_end, uint64_t* launches) {
  if (!h) return fail(nullptr, MLPV_E_INVALID, "handle is NULL");
  h->ev_begin = static_cast<cudaEvent_t>(ev_begin);
  h->ev_end = static_cast<cudaEvent_t>(ev_end);
  if (launches) *launches = h->launches;
  return MLPV_OK;
}

// ---------------------------------------------------------------------------------------- entry points
extern "C" mlpv_status mlpv_coverage_layout(mlpv_t h, const mlpv_coverage_spec* cov, size_t* n_words, size_t* offs) {
  if (!h) return fail(nullptr, MLPV_E_INVALID, "handle is NULL");
  DevCov dc;
  mlpv_status s = build_cov(h, cov, &dc);
  if (s != MLPV_OK) return s;
  if (n_words) *n_words = dc.n_words;
  if (offs)
    for (int p = 0; p < dc.n_pairs; p++)
      for (int m = 0; m < 4; m++) offs[4 * p + m] = dc.off[p][m];
  return MLPV_OK;
}

extern "C" mlpv_status mlpv_space_size(mlpv_t h, const mlpv_pert* pert, uint64_t* size) {
  if (!h || !size) return fail(h, MLPV_E_INVALID, "handle or size is NULL");
  DevPert dp;
  mlpv_status s = build_pert(h, pert, &dp, false);
  if (s != MLPV_OK) return s;
  *size = space_of(h->net, pert);
  return MLPV_OK;
}

static mlpv_status check_impl(mlpv_t h, const void* base_inputs, int32_t n_base, const mlpv_pert* pert,
                              const mlpv_property* prop, const mlpv_coverage_spec* cov, const mlpv_result* res,
                              void* stream, const mlpv_incremental* inc, int32_t* step, int32_t* step_u);

extern "C" mlpv_status mlpv_check(mlpv_t h, const void* base_inputs, int32_t n_base, const mlpv_pert* pert,
                                  const mlpv_property* prop, const mlpv_coverage_spec* cov, const mlpv_result* res,
                                  void* stream) {
  return check_impl(h, base_inputs, n_base, pert, prop, cov, res, stream, nullptr, nullptr, nullptr);
}

// Incremental bounds (reading C28): one enumeration of
// the gamma ball whose first-counterexample keys carry the step of the smallest ball b_i holding
// the candidate; the iteration-by-iteration loop of the paper reports the same (step, index).
extern "C" mlpv_status mlpv_check_incremental(mlpv_t h, const void* base_inputs, int32_t n_base, const mlpv_pert* pert,
                                              const mlpv_property* prop, const mlpv_coverage_spec* cov,
                                              const mlpv_incremental* inc, const mlpv_result* res, int32_t* step,
                                              int32_t* step_unflagged, void* stream) {
  if (!h) return fail(nullptr, MLPV_E_INVALID, "handle is NULL");
  if (!inc || !step || !step_unflagged) return fail(h, MLPV_E_INVALID, "inc / step / step_unflagged is NULL");
  return check_impl(h, base_inputs, n_base, pert, prop, cov, res, stream, inc, step, step_unflagged);
}

extern "C" double mlpv_incremental_bound(const mlpv_incremental* inc, int32_t i) {
  if (!inc || inc->max_bound < 1 || inc->granularity < 1) return 0.0;
  const int64_t ig = (int64_t)i * inc->granularity;
  if (ig >= inc->max_bound) return inc->gamma;
  return (double)ig * (inc->gamma / (double)inc->max_bound);
}

extern "C" int32_t mlpv_incremental_steps(const mlpv_incremental* inc) {
  if (!inc || inc->max_bound < 1 || inc->granularity < 1) return 0;
  return (int32_t)((inc->max_bound + inc->granularity - 1) / inc->granularity);
}

static mlpv_status check_impl(mlpv_t h, const void* base_inputs, int32_t n_base, const mlpv_pert* pert,
                              const mlpv_property* prop, const mlpv_coverage_spec* cov, const mlpv_result* res,
                              void* stream, const mlpv_incremental* inc, int32_t* step, int32_t* step_u) {
  if (!h) return fail(nullptr, MLPV_E_INVALID, "handle is NULL");
  if (h->sticky != MLPV_OK) return fail(h, h->sticky, "handle has a sticky CUDA error: %s", h->err.c_str());
  if (!base_inputs || n_base < 1) return fail(h, MLPV_E_INVALID, "base_inputs is NULL or n_base = %d", n_base);
  if (!res || !res->checked || !res->violated || !res->flagged || !res->first_cex || !res->first_cex_unflagged)
    return fail(h, MLPV_E_INVALID, "result buffers are NULL");
  DevPert dp; DevProp dprop; DevCov dc;
  mlpv_status s;
  if ((s = build_pert(h, pert, &dp, true)) != MLPV_OK) return s;
  if ((s = build_prop(h, prop, &dprop)) != MLPV_OK) return s;
  if ((s = build_cov(h, cov, &dc)) != MLPV_OK) return s;
  if (dc.n_words > 0 && (!res->cov_all || !res->cov_certain)) return fail(h, MLPV_E_INVALID, "coverage result buffers are NULL");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_TRY(h, cudaSetDevice(h->device), "cudaSetDevice");
  mlpv_pert pinc;
  if (inc) {
    if (!(inc->gamma > 0) || !std::isfinite(inc->gamma)) return fail(h, MLPV_E_INVALID, "inc.gamma = %g (finite, > 0)", inc->gamma);
    if (inc->max_bound < 1 || inc->granularity < 1) return fail(h, MLPV_E_INVALID, "inc.max_bound / granularity must be >= 1");
    if ((inc->early_exit != 0 && inc->early_exit != 1) || inc->reserved != 0)
      return fail(h, MLPV_E_INVALID, "inc.early_exit = %d (0 or 1), inc.reserved = %d (0)", inc->early_exit, inc->reserved);
    const int n_steps = mlpv_incremental_steps(inc);
    if (n_steps > kMaxSteps) return fail(h, MLPV_E_INVALID, "inc: %d steps (max %d)", n_steps, kMaxSteps);
    if (is_philox(pert->kind))
      return fail(h, MLPV_E_UNSUPPORTED, "incremental bounds are built for the subset and tuple spaces");
    if (pert->index_end > (1ull << kStepShift)) return fail(h, MLPV_E_UNSUPPORTED, "incremental bounds need index_end <= 2^48");
    pinc = *pert;
    pinc.restrict_l2 = inc->gamma;               // the kernel enumerates the whole gamma ball once
    pert = &pinc;
    if ((s = build_pert(h, pert, &dp, true)) != MLPV_OK) return s;
    std::vector<double> r2f(n_steps);
    std::vector<long long> r2i(n_steps);
    const bool fx = is_fixed(h->net.numeric);
    const double S = h->net.numeric == MLPV_NUM_Q4_12 ? 4096.0 : 255.0;
    for (int i = 1; i <= n_steps; i++) {
      const double b = mlpv_incremental_bound(inc, i);
      r2f[i - 1] = b * b;
      r2i[i - 1] = (long long)std::floor(b * b * S * S);
    }
    // pageable source: cudaMemcpyAsync returns once the data is staged
    CUDA_TRY(h, cudaMemcpyAsync(h->steps_dev, fx ? (const void*)r2i.data() : (const void*)r2f.data(), 8ull * n_steps,
                                cudaMemcpyHostToDevice, st), "copy steps");
    dp.n_steps = n_steps;
    dp.step_r2_f = static_cast<const double*>(h->steps_dev);
    dp.step_r2_raw = static_cast<const long long*>(h->steps_dev);
  }
  DevResult dr{res->checked, res->violated, res->flagged, res->first_cex, res->first_cex_unflagged, res->cov_all, res->cov_certain};
  CUDA_TRY(h, launch_init_result(dr, n_base, dc.n_words, st), "init results");
  h->launches++;
  Plan plan;
  const bool fl = !is_fixed(h->net.numeric);
  if ((s = prepare(h, base_inputs, n_base, pert, dp, &dc, &plan, st, fl)) != MLPV_OK) return s;
  dc.tau_dev = (fl && !cov->tau) ? plan.tau_dev : nullptr;
  if (pert->index_begin != pert->index_end && is_philox(pert->kind) && dp.restrict_on) {
    // restriction R on a Philox space: per chunk of the range, the mask pass marks the candidates
    // inside R, then the enumeration kernel checks the marked ones (results accumulate over chunks)
    const uint64_t len = pert->index_end - pert->index_begin;
    uint64_t chunk = ((uint64_t)1 << 31) / (uint64_t)n_base;        // <= 256 MB of mask bits per pass
    chunk = chunk < 32 ? 32 : chunk & ~(uint64_t)31;
    if (chunk > len) chunk = len;
    const uint32_t wpb = (uint32_t)((chunk + 31) / 32);
    void* mask = nullptr;
    CUDA_TRY(h, cudaMallocAsync(&mask, 4ull * wpb * n_base, st), "restriction mask");
    mlpv_status rs = MLPV_OK;
    for (uint64_t b0 = pert->index_begin; b0 < pert->index_end && rs == MLPV_OK; b0 += chunk) {
      mlpv_pert pc = *pert;
      pc.index_begin = b0;
      pc.index_end = b0 + chunk < pert->index_end ? b0 + chunk : pert->index_end;
      DevPert dpc = dp;
      dpc.begin = pc.index_begin;
      dpc.end = pc.index_end;
      dpc.rmask = static_cast<const uint32_t*>(mask);
      dpc.rmask_begin = pc.index_begin;
      dpc.rmask_wpb = wpb;
      cudaError_t e = launch_restrict_mask(h->net, base_inputs, n_base, dpc, static_cast<uint32_t*>(mask), st);
      if (e != cudaSuccess) { rs = cuda_fail(h, e, "restriction mask"); break; }
      h->launches++;
      rs = run_kernel(h, base_inputs, n_base, &pc, dpc, dprop, dc, dr, plan, nullptr, 0, 0, nullptr, st);
    }
    cudaFreeAsync(mask, st);
    if (rs != MLPV_OK) return rs;
  } else if (pert->index_begin != pert->index_end && inc && inc->early_exit) {
    // the loop's own order (NEXT-2 early exit): pass i checks the shell
    // b_(i-1) < delta <= b_i of the base inputs not decided by passes 1 .. i-1 (the unflagged keys
    // in first_cex_unflagged, stream-ordered); a decided base's blocks return at once, so the
    // passes after the last decision cost a launch each and no host synchronisation is needed
    dp.decided = reinterpret_cast<const unsigned long long*>(dr.first_cex_unflagged);
    const cudaEvent_t ev0 = h->ev_begin;              // mlpv_profile brackets all the passes
    for (int i = 1; i <= dp.n_steps && s == MLPV_OK; i++) {
      dp.shell = i;
      s = run_kernel(h, base_inputs, n_base, pert, dp, dprop, dc, dr, plan, nullptr, 0, 0, nullptr, st);
      h->ev_begin = nullptr;
    }
    h->ev_begin = ev0;
    if (s != MLPV_OK) return s;
  } else if (pert->index_begin != pert->index_end) {
    if ((s = run_kernel(h, base_inputs, n_base, pert, dp, dprop, dc, dr, plan, nullptr, 0, 0, nullptr, st)) != MLPV_OK)
      return s;
  }
  if (inc) {
    CUDA_TRY(h, launch_split_steps(dr, n_base, step, step_u, st), "split steps");
    h->launches++;
  }
  return MLPV_OK;
}

extern "C" mlpv_status mlpv_eval(mlpv_t h, const void* base_inputs, int32_t n_base, int32_t base_id,
                                 const mlpv_pert* pert, const uint64_t* indices, int64_t n, void* out, void* stream) {
  if (!h) return fail(nullptr, MLPV_E_INVALID, "handle is NULL");
  if (h->sticky != MLPV_OK) return fail(h, h->sticky, "handle has a sticky CUDA error: %s", h->err.c_str());
  if (!base_inputs || n_base < 1 || base_id < 0 || base_id >= n_base) return fail(h, MLPV_E_INVALID, "base_inputs / n_base / base_id");
  if (n < 0 || (n > 0 && (!indices || !out))) return fail(h, MLPV_E_INVALID, "indices / out / n");
  DevPert dp;
  mlpv_status s;
  if ((s = build_pert(h, pert, &dp, false)) != MLPV_OK) return s;
  if (n == 0) return MLPV_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_TRY(h, cudaSetDevice(h->device), "cudaSetDevice");
  DevCov dc;
  memset(&dc, 0, sizeof dc);
  DevProp dprop;
  memset(&dprop, 0, sizeof dprop);
  DevResult dr{};
  Plan plan;
  if ((s = prepare(h, base_inputs, n_base, pert, dp, &dc, &plan, st, false)) != MLPV_OK) return s;
  return run_kernel(h, base_inputs, n_base, pert, dp, dprop, dc, dr, plan, indices, n, base_id, out, st);
}

// Host-side candidate reconstruction (the product's own decoder; reading C14).
static uint32_t mulhi32(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * b) >> 32); }
static void philox_host(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; r++) {
    const uint32_t h0 = mulhi32(0xD2511F53u, c[0]), l0 = 0xD2511F53u * c[0];
    const uint32_t h1 = mulhi32(0xCD9E8D57u, c[2]), l1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = h1 ^ c[1] ^ k0, n2 = h0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = l1; c[2] = n2; c[3] = l0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
}
static uint16_t f2bf_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

extern "C" mlpv_status mlpv_decode(mlpv_numeric numeric, const mlpv_pert* p, const void* base, int32_t n0, int32_t base_id,
                                   uint64_t index, void* out) {
  if (!p || !base || !out || n0 < 1) return fail(nullptr, MLPV_E_INVALID, "pert / base / out / n_0");
  const size_t es = in_elem(numeric);
  memcpy(out, base, es * (size_t)n0);
  auto set = [&](int j, double v) {
    switch (numeric) {
      case MLPV_NUM_FP32: static_cast<float*>(out)[j] = (float)v; break;
      case MLPV_NUM_BF16: static_cast<uint16_t*>(out)[j] = f2bf_rne((float)v); break;
      case MLPV_NUM_Q4_12: static_cast<int16_t*>(out)[j] = (int16_t)v; break;
      default: static_cast<uint8_t*>(out)[j] = (uint8_t)v; break;
    }
  };
  auto get = [&](const void* a, int j) -> double {
    switch (numeric) {
      case MLPV_NUM_FP32: return static_cast<const float*>(a)[j];
      case MLPV_NUM_BF16: return bf16_to_double(static_cast<const uint16_t*>(a)[j]);
      case MLPV_NUM_Q4_12: return static_cast<const int16_t*>(a)[j];
      default: return static_cast<const uint8_t*>(a)[j];
    }
  };
  auto lvl = [&](int q) -> double {
    if (numeric == MLPV_NUM_FP32) return static_cast<const float*>(p->levels)[q];
    if (numeric == MLPV_NUM_BF16) return bf16_to_double(static_cast<const uint16_t*>(p->levels)[q]);
    return static_cast<const int16_t*>(p->levels)[q];
  };
  const uint64_t q = (uint64_t)p->n_levels;
  if (p->kind == MLPV_PERT_TUPLE_REPLACE) {
    if (p->tuple == 1) { set((int)(index / q), lvl((int)(index % q))); return MLPV_OK; }
    uint64_t pr = index / (q * q);
    const uint64_t rem = index % (q * q);
    int i = 0;
    while (pr >= (uint64_t)(n0 - 1 - i)) { pr -= (uint64_t)(n0 - 1 - i); i++; }
    set(i, lvl((int)(rem / q)));
    set(i + 1 + (int)pr, lvl((int)(rem % q)));
    return MLPV_OK;
  }
  if (p->kind == MLPV_PERT_SUBSET_OFFSET || p->kind == MLPV_PERT_SUBSET_REPLACE) {
    uint64_t c = index;
    for (int k = p->n_pixels - 1; k >= 0; k--) {
      const int d = (int)(c % q);
      c /= q;
      const int px = p->pixels[k];
      if (p->kind == MLPV_PERT_SUBSET_REPLACE) set(px, lvl(d));
      else {
        const double hi = numeric == MLPV_NUM_Q4_12 ? 4096 : 255;
        double v = get(base, px) + lvl(d);
        set(px, v < 0 ? 0 : (v > hi ? hi : v));
      }
    }
    return MLPV_OK;
  }
  const uint32_t k0 = (uint32_t)p->seed, k1 = (uint32_t)(p->seed >> 32);
  if (p->kind == MLPV_PERT_PHILOX_BOX || p->kind == MLPV_PERT_PHILOX_CLAMP) {   // exact real candidate (doubles)
    double* o = static_cast<double*>(out);
    for (int j = 0; j < n0; j++) o[j] = get(base, j);
    for (int j = 0; j < (n0 + 31) / 32; j++) {
      uint32_t w[4] = {(uint32_t)index, (uint32_t)(index >> 32), (uint32_t)base_id, (uint32_t)j};
      philox_host(w, k0, k1);
      for (int ww = 0; ww < 4; ww++)
        for (int nb = 0; nb < 8; nb++) {
          const int px = 32 * j + 8 * ww + nb;
          if (px >= n0) continue;
          double v = o[px] + (p->lattice_origin + (double)((w[ww] >> (4 * nb)) & 15) * p->lattice_step);
          if (p->kind == MLPV_PERT_PHILOX_CLAMP) v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
          o[px] = v;
        }
    }
    return MLPV_OK;
  }
  for (int j = 0; j < (n0 + 31) / 32; j++) {
    uint32_t w[4] = {(uint32_t)index, (uint32_t)(index >> 32), (uint32_t)base_id, (uint32_t)j};
    philox_host(w, k0, k1);
    for (int ww = 0; ww < 4; ww++)
      for (int nb = 0; nb < 8; nb++) {
        const int px = 32 * j + 8 * ww + nb;
        if (px >= n0) continue;
        const int l = (w[ww] >> (4 * nb)) & 15;
        if (numeric == MLPV_NUM_BF16) {
          // off = RNE_bf16(l*step + origin) (exact in fp32), x + off exact in fp64, clamp, RNE
          const float off = bf16_to_double(f2bf_rne((float)(l * p->lattice_step + p->lattice_origin)));
          double v = get(base, px) + (double)off;
          v = v < 0 ? 0 : (v > 1 ? 1 : v);
          // round the exact double to bf16 via fp32 only when exact in fp32; otherwise split
          float vf = (float)v;
          if ((double)vf != v) {
            // nearest bf16 of v: compare the two bf16 neighbours of the truncation
            uint32_t u; memcpy(&u, &vf, 4);
            float lo, hi;
            uint32_t t = u & 0xFFFF0000u; memcpy(&lo, &t, 4);
            t += 0x10000u; memcpy(&hi, &t, 4);
            if (lo > v) { hi = lo; t = (u & 0xFFFF0000u) - 0x10000u; memcpy(&lo, &t, 4); }
            const double dl = v - lo, dh = hi - v;
            uint32_t ul; memcpy(&ul, &lo, 4);
            vf = (dl < dh || (dl == dh && ((ul >> 16) & 1u) == 0)) ? lo : hi;
            static_cast<uint16_t*>(out)[px] = (uint16_t)(*reinterpret_cast<uint32_t*>(&vf) >> 16);
          } else {
            static_cast<uint16_t*>(out)[px] = f2bf_rne(vf);
          }
        } else {
          double v = get(base, px) + (double)l * p->lattice_step + p->lattice_origin;
          set(px, v < 0 ? 0 : (v > 255 ? 255 : v));
        }
      }
  }
  return MLPV_OK;
}

extern "C" mlpv_status mlpv_sync(mlpv_t h, void* stream) {
  if (!h) return fail(nullptr, MLPV_E_INVALID, "handle is NULL");
  if (h->sticky != MLPV_OK) return fail(h, h->sticky, "handle has a sticky CUDA error: %s", h->err.c_str());
  CUDA_TRY(h, cudaSetDevice(h->device), "cudaSetDevice");
  CUDA_TRY(h, cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "asynchronous kernel fault");
  uint32_t st = 0;
  CUDA_TRY(h, cudaMemcpy(&st, h->dev_status, 4, cudaMemcpyDeviceToHost), "status read");
  if (st != 0) {
    CUDA_TRY(h, cudaMemset(h->dev_status, 0, 4), "status reset");
    if (st & kStatusQ412Base)
      return fail(h, MLPV_E_INVALID, "Q4_12: a base input pixel is outside the normalised raw range [0, 4096] "
                                     "(reading C16; the accumulator bound of mlpv_create assumes it); results not exact");
    if (st & kStatusClampBase)
      return fail(h, MLPV_E_INVALID, "PHILOX_CLAMP: a base pixel is outside [0, 1] or its binding clamp bound is not "
                                     "exactly representable at the contraction scale (mlpv.h); those results are not exact");
    return fail(h, MLPV_E_INVALID, "device status 0x%x", st);
  }
  return MLPV_OK;
}

extern "C" mlpv_status mlpv_merge(const mlpv_result* parts, int32_t n_parts, int32_t n_base, size_t n_words,
                                  const mlpv_result* out, void* stream) {
  if (!parts || !out || n_parts < 1 || n_parts > kMaxParts || n_base < 1)
    return fail(nullptr, MLPV_E_INVALID, "mlpv_merge: parts / out / n_parts (1..%d) / n_base", kMaxParts);
  MergeParts mp;
  memset(&mp, 0, sizeof mp);
  for (int i = 0; i < n_parts; i++)
    mp.p[i] = DevResult{parts[i].checked, parts[i].violated, parts[i].flagged, parts[i].first_cex,
                        parts[i].first_cex_unflagged, parts[i].cov_all, parts[i].cov_certain};
  DevResult o{out->checked, out->violated, out->flagged, out->first_cex, out->first_cex_unflagged, out->cov_all, out->cov_certain};
  cudaError_t e = launch_merge(mp, n_parts, n_base, n_words, o, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(nullptr, MLPV_E_CUDA, "merge: %s", cudaGetErrorString(e));
  return MLPV_OK;
}

extern "C" mlpv_status mlpv_pair_coverage(mlpv_t h, const void* images, int32_t n_images, const mlpv_coverage_spec* cov,
                                          uint32_t* cov_all, uint32_t* cov_certain, void* stream) {
  if (!h) return fail(nullptr, MLPV_E_INVALID, "handle is NULL");
  if (h->sticky != MLPV_OK) return fail(h, h->sticky, "handle has a sticky CUDA error: %s", h->err.c_str());
  if (!images || n_images < 1) return fail(h, MLPV_E_INVALID, "images is NULL or n_images = %d", n_images);
  DevCov dc;
  mlpv_status s = build_cov(h, cov, &dc);
  if (s != MLPV_OK) return s;
  if (dc.n_words > 0 && (!cov_all || !cov_certain)) return fail(h, MLPV_E_INVALID, "cov_all / cov_certain is NULL");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_TRY(h, cudaSetDevice(h->device), "cudaSetDevice");
  const DevNet& n = h->net;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t o_cls = al(4ull * n_images * n.trace_len), o_tau = o_cls + al(4ull * n_images);
  if ((s = ensure_ws(h, o_tau + al(4 * kMaxL), st)) != MLPV_OK) return s;
  char* w = static_cast<char*>(h->ws);
  BaseWS ws{};
  ws.trace = w;
  ws.cls = reinterpret_cast<int32_t*>(w + o_cls);
  DevPert dp;
  memset(&dp, 0, sizeof dp);
  dp.kind = MLPV_PERT_SUBSET_REPLACE;            // no delta table / box base (ws.delta, ws.base1 NULL)
  CUDA_TRY(h, launch_base_prologue(n, images, n_images, dp, nullptr, ws, st), "image traces");
  h->launches++;
  const bool fl = !is_fixed(n.numeric);
  if (fl && !cov->tau && dc.n_words > 0) {
    float* tau_dev = reinterpret_cast<float*>(w + o_tau);
    CUDA_TRY(h, launch_tau(n, ws.trace, n_images, tau_dev, st), "tau");
    h->launches++;
    dc.tau_dev = tau_dev;
  }
  if (dc.n_words == 0) return MLPV_OK;
  CUDA_TRY(h, launch_pair_cov(n, dc, ws.trace, n_images, cov_all, cov_certain, st), "pair coverage");
  h->launches++;
  return MLPV_OK;
}

extern "C" mlpv_status mlpv_neuron_coverage(mlpv_t h, const mlpv_coverage_spec* cov, const uint32_t* words,
                                            uint8_t* covered, uint32_t* counts, void* stream) {
  if (!h) return fail(nullptr, MLPV_E_INVALID, "handle is NULL");
  if (!words || !covered || !counts) return fail(h, MLPV_E_INVALID, "words / covered / counts is NULL");
  DevCov dc;
  mlpv_status s = build_cov(h, cov, &dc);
  if (s != MLPV_OK) return s;
  CUDA_TRY(h, cudaSetDevice(h->device), "cudaSetDevice");
  CUDA_TRY(h, launch_neuron_cov(h->net, dc, words, covered, counts, static_cast<cudaStream_t>(stream)), "neuron coverage");
  return MLPV_OK;
}
