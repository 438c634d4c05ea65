/*
 * mlpv.h -- C ABI of the B200-native MLP safety checker (arXiv 1907.12933, data-parallel core).
 *
 * The paper checks, symbolically, (a) the four covering methods SS / DS / SV / DV between pairs
 * of inputs (§III.B) and (b) `checkNN`: whether an image within a proximity
 * bound of a dataset image changes the classification (§III.C).  `checkNN`
 * takes "an ANN with its weights and bias descriptions", "the image to be checked" and "a
 * parameter that limits the proximity".  This library replaces the symbolic
 * search by exhaustive enumeration (or Philox sampling) of a discretised perturbation space
 * around each base image, evaluated on the GPU: for every candidate it runs the MLP forward pass
 * (Eq. 1-2), takes the argmax, tests the safety property
 * and accumulates SS / VS / SV / VV pair coverage between adjacent layers, base versus candidate.
 * The paper's DS-Cover is called VS here and DV-Cover is called VV.
 *
 * Conventions for every entry point:
 *   - all functions return mlpv_status; no exception crosses the ABI;
 *   - argument errors are detected synchronously, before any GPU work, and described by
 *     mlpv_last_error(handle) (mlpv_last_error(NULL) for errors of mlpv_create / mlpv_decode);
 *   - a CUDA failure is sticky: the handle reports MLPV_E_CUDA from then on;
 *   - a handle is bound to one device and is not thread-safe (one host thread at a time); its
 *     workspace and activation scratch are per handle, so the calls of one handle must be ordered
 *     on the device as well: use one stream per handle, or order its streams with events
 *     (independent handles may run concurrently on different streams);
 *   - "device" pointers are CUDA global-memory pointers on the handle's device; "host" pointers
 *     are ordinary process memory; `stream` is a cudaStream_t (NULL = legacy default stream).
 *
 * Numerics (readings C16-C19):
 *   MLPV_NUM_FP32  fp32 weights / inputs, fp32 biases, sigmoid or ReLU hidden layers, fp32 math.
 *   MLPV_NUM_BF16  bf16 weights / inputs, fp32 biases, ReLU hidden layers; tensor-core contraction
 *                  with fp32 accumulation; hidden activations carried at ~fp32 precision.
 *   MLPV_NUM_Q4_12 int16 Q4.12 weights / inputs, int32 Q8.24 accumulators and biases, hidden
 *                  requant u16 = sat16((acc + 2^11) >> 12), PL-sigmoid or ReLU; bit-exact.
 *   MLPV_NUM_INT8  int8 weights, u8 inputs, int32 accumulators and biases, hidden
 *                  y = min(255, max(0, (acc + 2^(sh-1)) >> sh)) (ReLU + requant); bit-exact.
 * Potentials ("u", the pre-activation of Eq. 1; for the output layer, the logits) are what every
 * predicate reads (reading C1).  Fixed-point potentials are int32 accumulators.
 */
#ifndef MLPV_H
#define MLPV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLPV_MAX_LAYERS 8      /* weight layers L */
#define MLPV_MAX_CLASSES 16    /* n_L */

typedef struct mlpv_ctx *mlpv_t;

typedef enum {
    MLPV_OK = 0,
    MLPV_E_INVALID = 1,      /* bad argument value (NULL pointer, out-of-range field, non-finite) */
    MLPV_E_SHAPE = 2,        /* inconsistent sizes */
    MLPV_E_UNSUPPORTED = 3,  /* valid but not built (numeric x activation x perturbation x shape) */
    MLPV_E_OVERFLOW = 4,     /* fixed-point worst-case accumulator bound >= 2^31 */
    MLPV_E_OOM = 5,          /* device allocation failed */
    MLPV_E_CUDA = 6          /* CUDA runtime / launch failure (sticky) */
} mlpv_status;

typedef enum { MLPV_NUM_FP32 = 0, MLPV_NUM_BF16 = 1, MLPV_NUM_Q4_12 = 2, MLPV_NUM_INT8 = 3 } mlpv_numeric;
typedef enum { MLPV_ACT_SIGMOID = 0, MLPV_ACT_PL_SIGMOID = 1, MLPV_ACT_RELU = 2 } mlpv_act;

/* The network ("weights and bias descriptions").  Host memory, read during
 * mlpv_create only (deep-copied to device memory owned by the handle).
 *   sizes[L+1]: n_0 (input pixels) .. n_L (classes, 1 <= n_L <= 16).
 *   W[l]: row-major n_{l+1} x n_l, element type by numeric: float | uint16 bf16 bits | int16 | int8.
 *   b[l]: n_{l+1} elements: float (FP32, BF16) | int32 in accumulator units (Q4_12, INT8). */
typedef struct {
    int32_t n_layers;
    const int32_t *sizes;
    const void *const *W;
    const void *const *b;
    mlpv_act hidden_act;
} mlpv_net;

/* Quantisation parameters (host, read during mlpv_create).
 *   requant_shift[L-1]: INT8 only, the per-hidden-layer shift sh_l >= 0 (reading C18).
 *   sigmoid_knots[129]: PL_SIGMOID only; Q4.12 knots over [-8, 8], step 1/8 (reading C17).
 *   acc_scale[L]: real value of one accumulator unit of layer l+1; used to convert the real
 *     thresholds of mlpv_coverage_spec / mlpv_property into accumulator units by round-to-nearest-
 *     even.  NULL means 1.0 (float numerics) or 2^-24 (Q4_12); required for INT8. */
typedef struct {
    mlpv_numeric numeric;
    const int32_t *requant_shift;
    const int16_t *sigmoid_knots;
    const double *acc_scale;
} mlpv_quant;

/* Perturbation spaces (reading C14; the discrete stand-in for the restriction R of
 * PAPER.md:453-461).  Index c of base input b names one candidate image:
 *   TUPLE_REPLACE  (tuple t = 1 or 2) pixels i<j ranked lexicographically (i outer), q levels:
 *                  c = rank(i,j) * q^2 + l_i * q + l_j;  x'_i = levels[l_i], x'_j = levels[l_j].
 *   SUBSET_OFFSET  K strictly ascending pixels P, q levels, P[0] most significant digit:
 *                  c = sum_k d_k q^(K-1-k);  x'_{P_k} = clamp(x_{P_k} + levels[d_k]) to [0, 4096]
 *                  (Q4_12) or [0, 255] (INT8).  Fixed-point numerics only.
 *   SUBSET_REPLACE as SUBSET_OFFSET with x'_{P_k} = levels[d_k].
 *   PHILOX_LATTICE every pixel p takes level l_p in [0,15]: for 32-pixel block j,
 *                  (w0..w3) = Philox4x32-10(counter = (c_lo, c_hi, b, j), key = (seed_lo, seed_hi)),
 *                  pixel 32j + 8w + n takes nibble n (LSB first) of word w.
 *                  BF16: x'_p = RNE_bf16(clamp(x_p + RNE_bf16(l_p*step + origin), 0, 1)), exact sums.
 *                  INT8: x'_p = clamp(x_p + l_p*step + origin, 0, 255), integer step / origin.
 *                  c < n_samples <= 2^32.  BF16 and INT8 numerics only.
 *   PHILOX_BOX     the same Philox levels, applied exactly: x'_p = x_p + origin + l_p * step as a
 *                  real number (no rounding to the input type, no clamping), i.e. the 16-point
 *                  lattice of the L-inf box [x - eps, x + eps] with origin = -eps, step = 2 eps / 15
 *                  (reading C14b).  Linear in the levels, so u_1 = W_1 x + b_1 +
 *                  origin W_1 1 + step W_1 l.  BF16 numerics, 3-layer nets with 256-wide hidden
 *                  layers (the k_fused3 path); other nets return MLPV_E_UNSUPPORTED.
 *                  mlpv_decode writes the candidate as n_0 doubles.
 *   PHILOX_CLAMP   the same Philox levels and box lattice, clamped to the image domain:
 *                  x'_p = min(max(x_p + origin + l_p * step, 0), 1) as a real number (reading C14:
 *                  "its values are normalized", §III.C; the candidate I lies in
 *                  M^{mn} of the restriction R).  BF16 numerics, base pixels
 *                  in [0, 1].  The tensor-core path (k_fused3: 3-layer nets with 256-wide hidden
 *                  layers, n_0 even, n_0 <= 1024) contracts d = x' - x = min(max(origin + l step,
 *                  -x), 1 - x) exactly in fp16 against W_1, which needs: every offset
 *                  (origin + l step) * 2^s and step * 2^(24+s) exactly representable in fp16 for
 *                  the library's scale s (MLPV_E_UNSUPPORTED otherwise; cfg4's step = 109 * 2^-14,
 *                  origin = -7.5 step qualify, s = -1), and every base pixel x = 0 or x * 2^s
 *                  representable (x >= 2^(-17-s)); a base image that breaks the last rule is
 *                  reported by mlpv_sync (MLPV_E_INVALID, the candidates' results are then not
 *                  exact).  mlpv_decode writes the candidate as n_0 doubles.
 * `levels` element type: float (FP32) | uint16 bf16 bits (BF16) | int16 (Q4_12, INT8).
 * Every call processes the half-open index range [index_begin, index_end) of EVERY base input;
 * disjoint ranges merge by sum / min / OR (mlpv_merge). */
typedef enum {
    MLPV_PERT_TUPLE_REPLACE = 0,
    MLPV_PERT_SUBSET_OFFSET = 1,
    MLPV_PERT_SUBSET_REPLACE = 2,
    MLPV_PERT_PHILOX_LATTICE = 3,
    MLPV_PERT_PHILOX_BOX = 4,
    MLPV_PERT_PHILOX_CLAMP = 5
} mlpv_pert_kind;

typedef struct {
    mlpv_pert_kind kind;
    int32_t tuple;
    int32_t n_pixels;
    const int32_t *pixels;       /* host */
    int32_t n_levels;
    const void *levels;          /* host */
    uint64_t seed;
    uint64_t n_samples;
    double lattice_step, lattice_origin;
    uint64_t index_begin, index_end;
    /* Restriction R of checkNN (reading C27): > 0 keeps only the
     * candidates I with delta(I^d, I) <= restrict_l2, the L2 distance to the base image in real
     * pixel units (FP32 / BF16 values, Q4.12 raw / 4096, INT8 raw / 255); the others are skipped
     * (not checked, no verdict, no coverage), so outside = range length - checked.  Fixed point:
     * sum of squared raw differences (int64) <= floor(restrict_l2^2 * S^2) in double, S = 4096 /
     * 255.  Float: sum over pixels, in pixel order, of (x' - x)^2 in double <= restrict_l2^2.
     * Every space: subset / tuple spaces filter inside the enumeration kernel (sum over the changed
     * pixels); the Philox spaces run a mask pass that rebuilds each candidate and sums over all
     * pixels in pixel order with separately rounded double operations (u8: exactly in integers).
     * 0 = no restriction. */
    double restrict_l2;
} mlpv_pert;

/* Safety property (reading C12).  Class = argmax of the logits, lowest index
 * on ties; the base class is the argmax of the base image's own forward pass.
 *   ARGMAX_UNCHANGED   violated iff class(x') != base class (the assert Y^d = N(I)).
 *   TARGET_NEVER       violated iff class(x') == target.
 *   THRESHOLD_LITERAL  violated iff y_D < V and y_i > V for some i != D (l_image_misclassified,
 *                      existential reading), D = target, or the base class if target < 0;
 *                      V in real units.
 *   THRESHOLD_LITERAL_ALL  the universal reading of the same literal (SURVEY
 *                      NEXT-4): violated iff y_D < V and y_i > V for every i != D.
 * Float numerics flag a candidate for the literal forms when some |y_i - V| < near_tie. */
typedef enum {
    MLPV_PROP_ARGMAX_UNCHANGED = 0,
    MLPV_PROP_TARGET_NEVER = 1,
    MLPV_PROP_THRESHOLD_LITERAL = 2,
    MLPV_PROP_THRESHOLD_LITERAL_ALL = 3
} mlpv_prop_kind;

typedef struct { mlpv_prop_kind kind; int32_t target; double V; } mlpv_property;

/* Coverage.  For each configured pair p = (k, k+1), 1 <= k < L:
 *   sc(n) = sign(u) != sign(u_base), sign(u) = [u >= 0];
 *   vc(n) = !sc(n) && |u - u_base| >= d_value;                  (reading C5)
 *   dc(k) = no sc in layer k && max_i |u - u_base| >= d_distance (reading C7, L-inf);
 *   SS(i,j) = sc(k,i) && exactly one sc in layer k && sc(k+1,j);  SV(i,j) likewise with vc(k+1,j);
 *   VS(j) = dc(k) && sc(k+1,j);  VV(j) = dc(k) && vc(k+1,j)   (column masks, reading C8).
 * Word layout per pair (mlpv_coverage_layout): SS [n_k * wpr] | SV [n_k * wpr] | VS [wpr] |
 * VV [wpr] uint32 words, wpr = ceil(n_{k+1} / 32), bit j of row i at word i*wpr + j/32, bit j%32.
 * Float numerics: near_tie is the top-2 logit margin below which a verdict is flagged (C20);
 * tau[L] (host, may be NULL = 1e-6 + 1e-5 * max|u_base| per layer, from this call's base
 * traces) is the predicate-ambiguity width: a candidate with a sign, value or distance predicate
 * of pair p within tau of its decision boundary contributes to cov_all only, not cov_certain. */
typedef struct {
    int32_t n_pairs;
    const int32_t *lower_layer;  /* host [n_pairs] */
    double d_value, d_distance;
    double near_tie;
    const double *tau;           /* host [L] or NULL */
} mlpv_coverage_spec;

/* Results: caller-allocated DEVICE buffers.  mlpv_check initialises them (counts 0, indices
 * UINT64_MAX = none, words 0) on `stream` before accumulating.  first_cex is the lowest violating
 * index of each base input's own space (reading C22).  Fixed-point numerics: flagged = 0,
 * first_cex_unflagged = first_cex, cov_certain = cov_all. */
typedef struct {
    uint64_t *checked, *violated, *flagged;      /* [n_base] */
    uint64_t *first_cex, *first_cex_unflagged;   /* [n_base] */
    uint32_t *cov_all, *cov_certain;             /* [n_words] (may be NULL if n_pairs == 0) */
} mlpv_result;

/* Create a handle on `device`: validates the net (sizes >= 1, 1 <= L <= 8, n_L <= 16, finite
 * values, numeric x activation built, fixed-point bound sum_j |w_j| x_max + |b| < 2^31 for every
 * neuron) and deep-copies it to device memory it owns.  Caller buffers may be freed on return. */
mlpv_status mlpv_create(const mlpv_net *net, const mlpv_quant *quant, int device, mlpv_t *out);

/* Frees the handle's device memory (synchronises the device first). NULL is a no-op. */
void mlpv_destroy(mlpv_t h);

/* Message of the last error on h (or of the last mlpv_create / mlpv_decode failure on this
 * thread if h == NULL); "" if none.  Owned by the library. */
const char *mlpv_last_error(mlpv_t h);

/* Coverage word count and per-pair word offsets (pair_offsets[4p + m], m = SS, SV, VS, VV). */
mlpv_status mlpv_coverage_layout(mlpv_t h, const mlpv_coverage_spec *cov, size_t *n_words,
                                 size_t *pair_offsets /* host [4 * n_pairs] or NULL */);

/* Size of one base input's index space. */
mlpv_status mlpv_space_size(mlpv_t h, const mlpv_pert *pert, uint64_t *size);

/* The check (the data-parallel checkNN + covering methods).  base_inputs: device
 * [n_base x n_0] in the input element type.  Enqueues all work on `stream` and returns without
 * synchronising.  Work = n_base * (index_end - index_begin) candidates. */
mlpv_status mlpv_check(mlpv_t h, const void *base_inputs, int32_t n_base, const mlpv_pert *pert,
                       const mlpv_property *prop, const mlpv_coverage_spec *cov,
                       const mlpv_result *res, void *stream);

/* Incremental bounds: the GPU analog of the two-step incremental BMC loop
 * (§II.B; SPEC.md incremental_verify).  Iteration i = 1, 2, .. checks the ball
 * delta(I^d, I) <= b_i (the restriction R of mlpv_pert.restrict_l2) and stops at the first
 * iteration with a counterexample (step one: violation) or when b_i = gamma (step two: the ball
 * is complete, the verdict is "safe over the grid").  Schedule (reading C28):
 *   Delta = gamma / max_bound,  b_i = (i g >= max_bound) ? gamma : (i g) * Delta   (double),
 *   i = 1 .. n_steps = ceil(max_bound / g);  g = granularity (the paper's increment, default 1;
 *   g > 1 may miss the nearest counterexample: PAPER.md:170-173). */
typedef struct {
    double gamma;          /* radius of the outer ball, finite > 0 (real pixel units as restrict_l2) */
    int32_t max_bound;     /* >= 1 */
    int32_t granularity;   /* >= 1 */
    int32_t early_exit;    /* 0: one enumeration of the gamma ball, keys (step, index);
                            * 1: the loop's own order with early exit: pass i
                            *    checks only the shell b_(i-1) < delta <= b_i of every base input not
                            *    yet decided (a base is decided once an unflagged violation is found),
                            *    so a base input's work stops at its counterexample's iteration */
    int32_t reserved;      /* 0 */
} mlpv_incremental;

/* n_steps of the schedule (0 if inc is NULL or invalid). */
int32_t mlpv_incremental_steps(const mlpv_incremental *inc);
/* b_i of the schedule, 1 <= i <= n_steps (the exact double both the library and a caller's loop
 * use); 0.0 if inc is NULL or invalid. */
double mlpv_incremental_bound(const mlpv_incremental *inc, int32_t i);

/* The incremental loop, per base input, in ONE enumeration of the gamma ball: step[b] (device
 * int32 [n_base]) = the first iteration i whose ball holds a violating candidate (0: none, i.e.
 * safe after n_steps iterations), first_cex[b] = the lowest index among the violating candidates
 * inside b_step -- what the loop reports at that iteration.  step_unflagged / first_cex_unflagged:
 * the same over unflagged violations (float numerics, reading C20).  The other result fields are
 * those of mlpv_check with restrict_l2 = gamma (pert->restrict_l2 is ignored) -- with early_exit = 1,
 * those of mlpv_check with restrict_l2 = b_(s_b) for each base input b, s_b = step_unflagged[b] if
 * nonzero else n_steps: the ball the paper's loop had checked when it stopped for b;
 * step / first_cex / step_unflagged / first_cex_unflagged are the same in both modes.  Subset / tuple
 * spaces with index_end <= 2^48 and n_steps <= 2048; MLPV_E_UNSUPPORTED otherwise.  Errors as
 * mlpv_check, plus MLPV_E_INVALID for a NULL / invalid inc or NULL step arrays. */
mlpv_status mlpv_check_incremental(mlpv_t h, const void *base_inputs, int32_t n_base, const mlpv_pert *pert,
                                   const mlpv_property *prop, const mlpv_coverage_spec *cov,
                                   const mlpv_incremental *inc, const mlpv_result *res, int32_t *step,
                                   int32_t *step_unflagged, void *stream);

/* Parity hook: potentials of every layer (layers 1..L concatenated, T = n_1 + .. + n_L values per
 * candidate) for candidates `indices` (device [n]) of base `base_id` of base_inputs (device
 * [n_base x n_0]), computed by the same kernels and arithmetic as mlpv_check.  out: device
 * [n x T], float (FP32, BF16) or int32 (Q4_12, INT8). */
mlpv_status mlpv_eval(mlpv_t h, const void *base_inputs, int32_t n_base, int32_t base_id,
                      const mlpv_pert *pert, const uint64_t *indices, int64_t n, void *out,
                      void *stream);

/* Counterexample reconstruction on the host: the candidate image `index` of base `base_id`
 * (base_input and image_out: host [n_0] in the input element type). */
mlpv_status mlpv_decode(mlpv_numeric numeric, const mlpv_pert *pert, const void *base_input,
                        int32_t n_0, int32_t base_id, uint64_t index, void *image_out);

/* Synchronise `stream` and report what the device found since the last call: MLPV_E_CUDA
 * (sticky) for an asynchronous kernel fault, MLPV_E_INVALID for an input error detected on the
 * device (a PHILOX_CLAMP base image that breaks its exactness rule; the status is then cleared).
 * mlpv_check / mlpv_eval never synchronise; a caller that reads results calls this first. */
mlpv_status mlpv_sync(mlpv_t h, void *stream);

/* Merge n_parts partial results of disjoint index ranges (device, laid out part-major:
 * counts [n_parts x n_base], words [n_parts x n_words]) into `out` by sum / min / OR on `stream`.
 * Used after the cross-GPU all-gather and for resumed sub-range runs. */
mlpv_status mlpv_merge(const mlpv_result *parts, int32_t n_parts, int32_t n_base, size_t n_words,
                       const mlpv_result *out, void *stream);

/* Dataset-pair coverage (PAPER.md:364-392 Eqs. sscover..dvcover and the
 * EG1 experiment): the four covers of every unordered pair {x_a, x_b}, a < b, of
 * an image set, OR-ed over all n_images (n_images - 1) / 2 pairs, in the word layout of
 * mlpv_coverage_layout (the same bit of a pair is set iff some pair of images covers it; x_a
 * takes the role the base has in mlpv_check, the covers being symmetric in the two images).
 * images: device [n_images x n_0] in the input element type.  cov_all / cov_certain: device
 * [n_words], overwritten (n_images = 1: all zero).  Float numerics: cov_certain holds the bits of
 * pairs none of whose predicates lies within tau of its boundary (reading C20; cov.tau NULL:
 * tau_l = 1e-6 + 1e-5 max over the images of max |u_l|); fixed point: cov_certain = cov_all.
 * The covered-neuron literal l_covered_neuron follows from mlpv_neuron_coverage on cov_all.
 * Uses the handle's workspace (4 (T + 1) n_images bytes); enqueued on `stream`, no sync.
 * Errors: MLPV_E_INVALID (NULL / n_images < 1 / bad spec), MLPV_E_OOM, MLPV_E_CUDA. */
mlpv_status mlpv_pair_coverage(mlpv_t h, const void *images, int32_t n_images, const mlpv_coverage_spec *cov,
                               uint32_t *cov_all, uint32_t *cov_certain, void *stream);

/* Neuron coverage (reading C9): covered[4 * T] bytes (device; method-major,
 * T = n_1 + .. + n_L, 1 = covered) and counts[4] (device uint32: covered neurons per method) from
 * the pair words.  A neuron is covered iff it is an endpoint of a covered pair; a VS / VV column j
 * covers every neuron of layer k and n_{k+1,j}. */
mlpv_status mlpv_neuron_coverage(mlpv_t h, const mlpv_coverage_spec *cov, const uint32_t *words,
                                 uint8_t *covered, uint32_t *counts, void *stream);

/* Measurement hook (bench.py): when ev_begin / ev_end (cudaEvent_t, or NULL to disable) are set,
 * subsequent mlpv_check calls record them on their stream immediately before and after the
 * enumeration kernel (k_small / k_large), so a caller can time that kernel alone.  *launches (may be
 * NULL) receives the number of kernels this handle has launched so far. */
mlpv_status mlpv_profile(mlpv_t h, void *ev_begin, void *ev_end, uint64_t *launches);

/* Library version string. */
const char *mlpv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MLPV_H */
