/*
 * mlpv_oracle.c -- plain, slow, obviously-correct CPU oracle for the MLP safety check.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  It shares no code, header, table or constant
 * generator with the CUDA path (paper_1907_12933_b200/), and includes nothing from include/.
 *
 * What it computes (brute force by the definition):
 *   for each base input b: full forward pass of the base image (all potentials, Eq. 1-2,
 *   PAPER.md:108-124), base class = argmax of the logits;
 *   for each index c of the requested range: decode the candidate image (readings C14/C15 in
 *   DESIGN.md), run the FULL forward pass with plain nested loops (no incremental layer 1, no
 *   tiling), evaluate sign / sc / vc / dc per neuron (§III.B), the four covering
 *   methods SS / DS(=VS) / SV / DV(=VV) on every configured layer pair,
 *   argmax and the safety property (§III.C), and accumulate counts, the
 *   lowest-index counterexample and the pair bitmaps.
 *
 * Arithmetic: fixed point (Q4.12, int8) in exact int64 with the rounding rules of readings C16-C18;
 * float (fp32, bf16 operands) evaluated in double on the exactly specified operands (C19), with
 * near-tie and predicate-ambiguity flags (C20).  Potentials of every numeric are held as doubles:
 * fixed-point accumulators are integers < 2^31 and therefore exact in double, so one predicate
 * implementation serves all numerics.
 *
 * Parity pins (tests/test_oracle_pins.py): Table I and Table II worked examples, closed-form
 * nets, the threshold net, brute force on tiny nets, library routines (numpy float64 matmul,
 * torch bf16 rounding, cuRAND Philox on the GPU).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { O_FP32 = 0, O_BF16 = 1, O_Q412 = 2, O_INT8 = 3 };
enum { O_SIGMOID = 0, O_PLSIG = 1, O_RELU = 2 };
enum { O_TUPLE = 0, O_SUB_OFF = 1, O_SUB_REP = 2, O_PHILOX = 3, O_BOX = 4, O_CLAMP = 5 };
enum { O_UNCHANGED = 0, O_TARGET = 1, O_LITERAL = 2, O_LITERAL_ALL = 3 };

typedef struct {
    int32_t L;
    const int32_t *sizes;     /* [L+1] */
    int32_t numeric;
    int32_t act;              /* hidden layers; the output layer has no activation */
    const void *const *W;     /* [L] row-major n_l x n_{l-1}: float | bf16 bits | int16 | int8 */
    const void *const *b;     /* [L] float (float numerics) | int32 accumulator units (fixed) */
    const int32_t *shift;     /* int8 requant shifts [L-1] */
    const int16_t *knots;     /* PL sigmoid: 129 Q4.12 knots */
    const double *acc_scale;  /* [L] real value of one accumulator unit */
} onet;

typedef struct {
    int32_t kind, tuple, n_pixels;
    const int32_t *pixels;
    int32_t n_levels;
    const void *levels;
    uint64_t seed, n_samples;
    double step, origin;
    uint64_t begin, end;
    double restrict_l2;       /* restriction R: > 0 keeps delta(I^d, I) <= restrict_l2 */
} opert;

typedef struct { int32_t kind, target; double V; } oprop;

typedef struct {
    int32_t n_pairs;
    const int32_t *lower;     /* pair p = (k, k+1) */
    double d_value, d_distance, near_tie;
    const double *tau;        /* [L] ambiguity widths (float numerics), tau[l-1] for layer l */
} ocov;

typedef struct {
    uint64_t *checked, *violated, *flagged, *first_cex, *first_cex_unflagged; /* [n_base] */
    uint32_t *cov_all, *cov_certain;                                          /* [n_words] */
} ores;

/* ------------------------------------------------------------------ numeric helpers */

/* bf16 bit pattern -> exact value */
static double bf16_val(uint16_t bits) {
    uint32_t u = (uint32_t)bits << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* Round a double to the nearest bf16 value (8 significant bits), ties to even.
 * Valid for the normal range, which is all this path produces. */
double orc_rne_bf16(double v) {
    if (v == 0.0 || !isfinite(v)) return v;
    int e;
    double m = frexp(v, &e);          /* v = m * 2^e, 0.5 <= |m| < 1 */
    double s = ldexp(m, 8);           /* 128 <= |s| < 256: the 8 kept bits are the integer part */
    double r = nearbyint(s);          /* default rounding mode: nearest, ties to even */
    return ldexp(r, e - 8);
}

/* floor(v / 2^s) for any sign (C16/C18 use arithmetic right shifts) */
static int64_t floor_shift(int64_t v, int s) {
    int64_t d = (int64_t)1 << s;
    int64_t q = v / d;                /* C division truncates toward zero */
    if ((v % d) != 0 && v < 0) q -= 1;
    return q;
}

static int64_t clamp64(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* C17 piecewise-linear sigmoid on a Q4.12 potential u16 in [-32768, 32767] */
int32_t orc_plsig(const int16_t *T, int32_t u16) {
    int32_t t = u16 + 32768;          /* 0 .. 65535 */
    int32_t i = t / 512, f = t % 512; /* segment, position within segment */
    int32_t y0 = T[i], y1 = T[i + 1];
    return y0 + (int32_t)floor_shift((int64_t)(y1 - y0) * f + 256, 9);
}

/* Philox4x32-10 (Salmon et al., SC'11; cuRAND's round function and constants, reading C15). */
void orc_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; r++) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static int is_fixed(int numeric) { return numeric == O_Q412 || numeric == O_INT8; }

static size_t elem_size(int numeric) {
    switch (numeric) { case O_FP32: return 4; case O_BF16: return 2; case O_Q412: return 2; default: return 1; }
}

/* value of input element j of an image stored in the numeric's input type:
 * float -> real value; fixed -> raw integer (as double, exact) */
static double in_get(int numeric, const void *img, int j) {
    switch (numeric) {
    case O_FP32: return (double)((const float *)img)[j];
    case O_BF16: return bf16_val(((const uint16_t *)img)[j]);
    case O_Q412: return (double)((const int16_t *)img)[j];
    default: return (double)((const uint8_t *)img)[j];
    }
}

static void in_set(int numeric, void *img, int j, double v) {
    switch (numeric) {
    case O_FP32: ((float *)img)[j] = (float)v; break;            /* v is already an fp32 value */
    case O_BF16: {                                                /* v is already a bf16 value */
        float f = (float)v; uint32_t u; memcpy(&u, &f, 4);
        ((uint16_t *)img)[j] = (uint16_t)(u >> 16); break; }
    case O_Q412: ((int16_t *)img)[j] = (int16_t)v; break;
    default: ((uint8_t *)img)[j] = (uint8_t)v; break;
    }
}

/* level q of the level array, in the same units as in_get */
static double level_get(int numeric, const void *lv, int q) {
    switch (numeric) {
    case O_FP32: return (double)((const float *)lv)[q];
    case O_BF16: return bf16_val(((const uint16_t *)lv)[q]);
    default: return (double)((const int16_t *)lv)[q];             /* Q4.12 raw / int8 values */
    }
}

static double w_get(const onet *n, int l, int i, int j) {          /* layer l (1-based) */
    int fan = n->sizes[l - 1];
    const void *W = n->W[l - 1];
    switch (n->numeric) {
    case O_FP32: return (double)((const float *)W)[(size_t)i * fan + j];
    case O_BF16: return bf16_val(((const uint16_t *)W)[(size_t)i * fan + j]);
    case O_Q412: return (double)((const int16_t *)W)[(size_t)i * fan + j];
    default: return (double)((const int8_t *)W)[(size_t)i * fan + j];
    }
}

/* ------------------------------------------------------------------ forward pass (Eq. 1-2) */

static int trace_len(const onet *n) {
    int t = 0;
    for (int l = 1; l <= n->L; l++) t += n->sizes[l];
    return t;
}

/* The net with every weight and bias converted once to its exact value as a double
 * (bf16 / int16 / int8 / int32 values are all exact in double). */
typedef struct { const onet *n; double *W[64]; double *b[64]; int maxw; } dnet;

static void dnet_init(dnet *d, const onet *n) {
    d->n = n; d->maxw = 0;
    for (int l = 0; l <= n->L; l++) if (n->sizes[l] > d->maxw) d->maxw = n->sizes[l];
    for (int l = 1; l <= n->L; l++) {
        int nl = n->sizes[l], fan = n->sizes[l - 1];
        d->W[l] = (double *)malloc(sizeof(double) * (size_t)nl * fan);
        d->b[l] = (double *)malloc(sizeof(double) * nl);
        for (int i = 0; i < nl; i++) {
            for (int j = 0; j < fan; j++) d->W[l][(size_t)i * fan + j] = w_get(n, l, i, j);
            d->b[l][i] = is_fixed(n->numeric) ? (double)((const int32_t *)n->b[l - 1])[i]
                                              : (double)((const float *)n->b[l - 1])[i];
        }
    }
}

static void dnet_free(dnet *d) {
    for (int l = 1; l <= d->n->L; l++) { free(d->W[l]); free(d->b[l]); }
}

/* potentials of layers 1..L, concatenated, into trace; h, hn: scratch of maxw doubles.
 * Returns 0, or -1 if a fixed-point accumulator leaves int32 (the C-ABI rejects such nets). */
static int forward_d(const dnet *d, const void *img, const double *ximg, double *trace, double *h, double *hn) {
    const onet *n = d->n;
    for (int j = 0; j < n->sizes[0]; j++) h[j] = ximg ? ximg[j] : in_get(n->numeric, img, j);
    int off = 0, rc = 0;
    for (int l = 1; l <= n->L; l++) {
        int nl = n->sizes[l], fan = n->sizes[l - 1];
        for (int i = 0; i < nl; i++) {
            const double *w = d->W[l] + (size_t)i * fan;
            double u;
            if (is_fixed(n->numeric)) {
                /* Eq. 1 in exact integer arithmetic */
                int64_t acc = (int64_t)d->b[l][i];
                for (int j = 0; j < fan; j++) acc += (int64_t)w[j] * (int64_t)h[j];
                if (acc > INT32_MAX || acc < INT32_MIN) rc = -1;
                u = (double)acc;
                if (l < n->L) {
                    if (n->numeric == O_Q412) {                 /* C16: Q8.24 -> Q4.12, round half up, sat */
                        int64_t u16 = clamp64(floor_shift(acc + 2048, 12), -32768, 32767);
                        if (n->act == O_PLSIG) hn[i] = (double)orc_plsig(n->knots, (int32_t)u16);
                        else hn[i] = (double)(u16 > 0 ? u16 : 0);             /* ReLU */
                    } else {                                    /* C18: ReLU + requant to u8 */
                        int sh = n->shift[l - 1];
                        int64_t r = sh > 0 ? ((int64_t)1 << (sh - 1)) : 0;
                        hn[i] = (double)clamp64(floor_shift(acc + r, sh), 0, 255);
                    }
                }
            } else {
                /* Eq. 1 on exact operands, evaluated in double (C19) */
                double s = 0.0;
                for (int j = 0; j < fan; j++) s += w[j] * h[j];
                u = s + d->b[l][i];
                if (l < n->L) {
                    if (n->act == O_SIGMOID) hn[i] = 1.0 / (1.0 + exp(-u));   /* Eq. 2 */
                    else hn[i] = u > 0.0 ? u : 0.0;                          /* ReLU */
                }
            }
            trace[off + i] = u;
        }
        off += nl;
        double *t = h; h = hn; hn = t;
    }
    return rc;
}

int orc_forward(const onet *n, const void *img, double *trace) {
    dnet d;
    dnet_init(&d, n);
    double *h = (double *)malloc(sizeof(double) * d.maxw), *hn = (double *)malloc(sizeof(double) * d.maxw);
    int rc = forward_d(&d, img, NULL, trace, h, hn);
    free(h); free(hn);
    dnet_free(&d);
    return rc;
}

/* ------------------------------------------------------------------ candidate decoding (C14) */

static uint64_t ipow(uint64_t b, int e) { uint64_t r = 1; while (e-- > 0) r *= b; return r; }

uint64_t orc_space_size(const opert *p, int n0) {
    if (p->kind == O_TUPLE) {
        uint64_t q = (uint64_t)p->n_levels;
        if (p->tuple == 1) return (uint64_t)n0 * q;
        return (uint64_t)n0 * (uint64_t)(n0 - 1) / 2 * q * q;
    }
    if (p->kind == O_SUB_OFF || p->kind == O_SUB_REP) return ipow((uint64_t)p->n_levels, p->n_pixels);
    return p->n_samples;
}

/* candidate `index` of base `base_id`: out = base with the perturbation applied */
void orc_decode(int numeric, const opert *p, const void *base, int n0, int base_id, uint64_t index, void *out) {
    memcpy(out, base, elem_size(numeric) * (size_t)n0);
    if (p->kind == O_TUPLE) {
        uint64_t q = (uint64_t)p->n_levels;
        if (p->tuple == 1) {
            int i = (int)(index / q);
            in_set(numeric, out, i, level_get(numeric, p->levels, (int)(index % q)));
            return;
        }
        uint64_t pr = index / (q * q), rem = index % (q * q);
        int li = (int)(rem / q), lj = (int)(rem % q);
        int i = 0;                    /* pairs i<j ranked lexicographically: i outer, j inner */
        while (pr >= (uint64_t)(n0 - 1 - i)) { pr -= (uint64_t)(n0 - 1 - i); i++; }
        int j = i + 1 + (int)pr;
        in_set(numeric, out, i, level_get(numeric, p->levels, li));
        in_set(numeric, out, j, level_get(numeric, p->levels, lj));
        return;
    }
    if (p->kind == O_SUB_OFF || p->kind == O_SUB_REP) {
        int K = p->n_pixels;
        uint64_t q = (uint64_t)p->n_levels, c = index;
        for (int k = K - 1; k >= 0; k--) {        /* P[0] is the most significant digit */
            int d = (int)(c % q); c /= q;
            int px = p->pixels[k];
            double v;
            if (p->kind == O_SUB_REP) v = level_get(numeric, p->levels, d);
            else {
                double hi = numeric == O_Q412 ? 4096.0 : 255.0;
                v = in_get(numeric, base, px) + level_get(numeric, p->levels, d);
                v = v < 0.0 ? 0.0 : (v > hi ? hi : v);
            }
            in_set(numeric, out, px, v);
        }
        return;
    }
    /* PHILOX_LATTICE: counter (s_lo, s_hi, b, j), key (seed_lo, seed_hi); pixel 32j+8w+n takes
     * nibble n (LSB first) of word w as level l in [0,15]. */
    uint32_t key[2] = { (uint32_t)p->seed, (uint32_t)(p->seed >> 32) };
    int nblk = (n0 + 31) / 32;
    for (int j = 0; j < nblk; j++) {
        uint32_t ctr[4] = { (uint32_t)index, (uint32_t)(index >> 32), (uint32_t)base_id, (uint32_t)j };
        uint32_t w[4];
        orc_philox(ctr, key, w);
        for (int ww = 0; ww < 4; ww++)
            for (int nb = 0; nb < 8; nb++) {
                int px = 32 * j + 8 * ww + nb;
                if (px >= n0) continue;
                int l = (int)((w[ww] >> (4 * nb)) & 15u);
                double x = in_get(numeric, base, px), v;
                if (numeric == O_BF16) {
                    double off = orc_rne_bf16((double)l * p->step + p->origin);   /* exact, then RNE */
                    v = x + off;                                                  /* exact in double */
                    v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
                    v = orc_rne_bf16(v);
                } else {                                                          /* u8 */
                    v = x + (double)l * p->step + p->origin;
                    v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
                }
                in_set(numeric, out, px, v);
            }
    }
}

/* PHILOX_BOX (reading C14b): the same Philox levels as PHILOX_LATTICE, applied exactly,
 * x'_p = x_p + origin + l_p * step as a real number (no rounding to the input type, no clamping):
 * the 16-point lattice of the L-inf box of radius -origin around x.
 * PHILOX_CLAMP (reading C14): the same point clamped to the image domain [0, 1],
 * x'_p = min(max(x_p + origin + l_p * step, 0), 1) -- the box lattice intersected with the
 * normalised images ("its values are normalized", §III.C; I in M^{mn},
 * PAPER.md:438, 454).  Both written as n0 doubles (exact for dyadic step / origin). */
void orc_decode_box(int numeric, const opert *p, const void *base, int n0, int base_id, uint64_t index, double *out) {
    uint32_t key[2] = { (uint32_t)p->seed, (uint32_t)(p->seed >> 32) };
    int nblk = (n0 + 31) / 32;
    for (int j = 0; j < nblk; j++) {
        uint32_t ctr[4] = { (uint32_t)index, (uint32_t)(index >> 32), (uint32_t)base_id, (uint32_t)j };
        uint32_t w[4];
        orc_philox(ctr, key, w);
        for (int ww = 0; ww < 4; ww++)
            for (int nb = 0; nb < 8; nb++) {
                int px = 32 * j + 8 * ww + nb;
                if (px >= n0) continue;
                int l = (int)((w[ww] >> (4 * nb)) & 15u);
                double v = in_get(numeric, base, px) + (p->origin + (double)l * p->step);
                if (p->kind == O_CLAMP) v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
                out[px] = v;
            }
    }
}

int orc_forward_dbl(const onet *n, const double *x, double *trace) {
    dnet d;
    dnet_init(&d, n);
    double *h = (double *)malloc(sizeof(double) * d.maxw), *hn = (double *)malloc(sizeof(double) * d.maxw);
    int rc = forward_d(&d, NULL, x, trace, h, hn);
    free(h); free(hn);
    dnet_free(&d);
    return rc;
}

/* ------------------------------------------------------------------ covering methods (§III.B) */

/* Coverage word layout per configured pair p = (k, k+1), n_k lower, n_{k+1} upper neurons,
 * wpr = ceil(n_{k+1}/32):  SS [n_k * wpr] | SV [n_k * wpr] | VS [wpr] | VV [wpr].
 * SS/SV rows are indexed by the lower neuron i, bit j by the upper neuron; VS/VV are column
 * masks (reading C8: the DS/DV condition does not involve i, so every i pairs with column j). */
size_t orc_coverage_layout(const int32_t *sizes, int n_pairs, const int32_t *lower, size_t *offs) {
    size_t w = 0;
    for (int p = 0; p < n_pairs; p++) {
        int k = lower[p];
        size_t wpr = (size_t)(sizes[k + 1] + 31) / 32;
        if (offs) {
            offs[4 * p + 0] = w;
            offs[4 * p + 1] = w + (size_t)sizes[k] * wpr;
            offs[4 * p + 2] = w + 2 * (size_t)sizes[k] * wpr;
            offs[4 * p + 3] = w + 2 * (size_t)sizes[k] * wpr + wpr;
        }
        w += 2 * (size_t)sizes[k] * wpr + 2 * wpr;
    }
    return w;
}

static int sign_of(double u) { return u >= 0.0 ? 1 : 0; }   /* 1 iff u >= 0 */

/* Evaluate the four covers for one pair of traces (t1 = x1, t2 = x2) and OR the covered pairs into
 * `words`.  dg[l-1] / dh[l-1]: value / distance thresholds of layer l in trace units.
 * If tau != NULL, *certain[p] reports whether no predicate used for pair p lies within tau of
 * its decision boundary (reading C20).
 *   sc(n)        = sign(u1) != sign(u2)
 *   vc(g, n)     = !sc(n) && |u2 - u1| >= d_g                              (C5)
 *   dc(h, k)     = no sc in layer k && max_i |u2 - u1| >= d_h              (C7)
 *   SS(i, j)     = sc(n_k,i) && no other sc in layer k && sc(n_k+1,j)      (C3)
 *   DS(., j)=VS  = dc(h, k) && sc(n_k+1,j)
 *   SV(i, j)     = sc(n_k,i) && no other sc in layer k && vc(g, n_k+1,j)
 *   DV(., j)=VV  = dc(h, k) && vc(g, n_k+1,j)  */
static void cover_eval(const int32_t *sizes, int L, const double *t1, const double *t2,
                       int n_pairs, const int32_t *lower, const double *dg, const double *dh,
                       const double *tau, uint32_t *words, int *certain) {
    int loff[64];
    loff[1] = 0;
    for (int l = 2; l <= L; l++) loff[l] = loff[l - 1] + sizes[l - 1];
    size_t w = 0;
    for (int p = 0; p < n_pairs; p++) {
        int k = lower[p], nk = sizes[k], nu = sizes[k + 1];
        size_t wpr = (size_t)(nu + 31) / 32;
        uint32_t *SS = words + w, *SV = SS + nk * wpr, *VS = SV + nk * wpr, *VV = VS + wpr;
        w += 2 * (size_t)nk * wpr + 2 * wpr;
        const double *a1 = t1 + loff[k], *a2 = t2 + loff[k];
        const double *b1 = t1 + loff[k + 1], *b2 = t2 + loff[k + 1];
        int n_sc = 0, i_star = -1;
        double linf = 0.0;
        int amb = 0;
        for (int i = 0; i < nk; i++) {
            if (sign_of(a1[i]) != sign_of(a2[i])) { n_sc++; if (i_star < 0) i_star = i; }
            double d = fabs(a2[i] - a1[i]);
            if (d > linf) linf = d;
            if (tau && (fabs(a1[i]) < tau[k - 1] || fabs(a2[i]) < tau[k - 1])) amb = 1;
        }
        int dc = (n_sc == 0) && (linf >= dh[k - 1]);
        if (tau && n_sc == 0 && fabs(linf - dh[k - 1]) < tau[k - 1]) amb = 1;
        for (int j = 0; j < nu; j++) {
            int sc = sign_of(b1[j]) != sign_of(b2[j]);
            double d = fabs(b2[j] - b1[j]);
            int vc = !sc && d >= dg[k];
            if (tau && (fabs(b1[j]) < tau[k] || fabs(b2[j]) < tau[k] || fabs(d - dg[k]) < tau[k])) amb = 1;
            uint32_t bit = 1u << (j % 32);
            size_t wj = (size_t)j / 32;
            if (n_sc == 1) {
                if (sc) SS[(size_t)i_star * wpr + wj] |= bit;
                if (vc) SV[(size_t)i_star * wpr + wj] |= bit;
            }
            if (dc) {
                if (sc) VS[wj] |= bit;
                if (vc) VV[wj] |= bit;
            }
        }
        if (certain) certain[p] = !amb;
    }
}

/* fixtures entry point: covers of two given traces (dg/dh per layer in trace units) */
void orc_cover(const int32_t *sizes, int L, const double *t1, const double *t2, int n_pairs,
               const int32_t *lower, const double *dg, const double *dh, uint32_t *words) {
    cover_eval(sizes, L, t1, t2, n_pairs, lower, dg, dh, NULL, words, NULL);
}

/* Same, with the ambiguity widths tau (reading C20): certain[p] = no predicate of pair p within
 * tau of its boundary.  Used by the dataset-pair workload. */
void orc_cover_tau(const int32_t *sizes, int L, const double *t1, const double *t2, int n_pairs,
                   const int32_t *lower, const double *dg, const double *dh, const double *tau,
                   uint32_t *words, int *certain) {
    cover_eval(sizes, L, t1, t2, n_pairs, lower, dg, dh, tau, words, certain);
}

/* ------------------------------------------------------------------ property (§III.C) */

/* argmax with lowest index on ties (reading C12) */
static int argmax_of(const double *y, int n) {
    int c = 0;
    for (int i = 1; i < n; i++) if (y[i] > y[c]) c = i;
    return c;
}

/* returns violated; *flag = near-tie / ambiguity flag (float numerics only) */
static int property_eval(const oprop *pr, const double *y, int n, int base_cls, double V,
                         int float_path, double near_tie, int *flag) {
    int cls = argmax_of(y, n);
    *flag = 0;
    if (pr->kind == O_LITERAL || pr->kind == O_LITERAL_ALL) {
        /* l_image_misclassified <=> (n_D < V) and (n_i > V) for some i != D (PAPER.md:487-489,
         * existential reading C12) or, O_LITERAL_ALL, for every i != D (the universal reading,
         * SURVEY NEXT-4); D = target, or the base class if target < 0 */
        int D = pr->target >= 0 ? pr->target : base_cls;
        int any = 0, all = 1;
        for (int i = 0; i < n; i++) {
            if (i != D && y[i] > V) any = 1;
            if (i != D && !(y[i] > V)) all = 0;
            if (float_path && fabs(y[i] - V) < near_tie) *flag = 1;
        }
        return (y[D] < V) && (pr->kind == O_LITERAL_ALL ? all : any);
    }
    if (float_path) {
        double top1 = y[cls], top2 = -INFINITY;
        for (int i = 0; i < n; i++) if (i != cls && y[i] > top2) top2 = y[i];
        if (n > 1 && top1 - top2 < near_tie) *flag = 1;
    }
    if (pr->kind == O_TARGET) return cls == pr->target;
    return cls != base_cls;                   /* safety assert Y^d = N(I) */
}

/* restriction R of checkNN (reading C27): delta(I^d, I) <= b with delta the L2
 * distance in real pixel units, by the definition: fixed point exactly in integers against
 * floor(b^2 S^2); float as the plain sum over all pixels of the squared differences in double */
static int within_restriction(int numeric, const void *base, const void *img, int n0, double b) {
    if (is_fixed(numeric)) {
        double S = numeric == O_Q412 ? 4096.0 : 255.0;
        int64_t thr = (int64_t)floor(b * b * S * S), s2 = 0;
        for (int p = 0; p < n0; p++) {
            int64_t d = (int64_t)in_get(numeric, img, p) - (int64_t)in_get(numeric, base, p);
            s2 += d * d;
        }
        return s2 <= thr;
    }
    double s2 = 0.0;
    for (int p = 0; p < n0; p++) {
        double d = in_get(numeric, img, p) - in_get(numeric, base, p);
        s2 += d * d;
    }
    return s2 <= b * b;
}

/* the same for a real-valued candidate (PHILOX_BOX / PHILOX_CLAMP): the sum over all pixels, in
 * pixel order, of (x'_p - x_p)^2 in double against b^2 */
static int within_restriction_real(int numeric, const void *base, const double *img, int n0, double b) {
    double s2 = 0.0;
    for (int p = 0; p < n0; p++) {
        double d = img[p] - in_get(numeric, base, p);
        s2 += d * d;
    }
    return s2 <= b * b;
}

/* ------------------------------------------------------------------ the check */

static double rne(double v) { return nearbyint(v); }

int orc_check(const onet *n, const void *bases, int n_base, const opert *p, const oprop *pr,
              const ocov *cov, ores *res, int nthreads) {
    int L = n->L, n0 = n->sizes[0], nL = n->sizes[L];
    int fl = !is_fixed(n->numeric);
    int T = trace_len(n);
    size_t nwords = orc_coverage_layout(n->sizes, cov->n_pairs, cov->lower, NULL);
    double dg[64], dh[64];
    for (int l = 1; l <= L; l++) {
        dg[l - 1] = fl ? cov->d_value : rne(cov->d_value / n->acc_scale[l - 1]);
        dh[l - 1] = fl ? cov->d_distance : rne(cov->d_distance / n->acc_scale[l - 1]);
    }
    double V = fl ? pr->V : rne(pr->V / n->acc_scale[L - 1]);
    memset(res->cov_all, 0, nwords * 4);
    memset(res->cov_certain, 0, nwords * 4);
    size_t esz = elem_size(n->numeric);
    int bad = 0;
    dnet dn;
    dnet_init(&dn, n);
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    for (int b = 0; b < n_base; b++) {
        const void *base = (const char *)bases + esz * (size_t)n0 * b;
        double *tb = (double *)malloc(sizeof(double) * T);
        {
            double *h = (double *)malloc(sizeof(double) * dn.maxw), *hn = (double *)malloc(sizeof(double) * dn.maxw);
            if (forward_d(&dn, base, NULL, tb, h, hn)) bad = 1;
            free(h); free(hn);
        }
        int base_cls = argmax_of(tb + T - nL, nL);
        uint64_t checked = 0, viol = 0, flg = 0, cex = UINT64_MAX, cexu = UINT64_MAX;
#pragma omp parallel
        {
            double *tc = (double *)malloc(sizeof(double) * T);
            double *h = (double *)malloc(sizeof(double) * dn.maxw), *hn = (double *)malloc(sizeof(double) * dn.maxw);
            void *img = malloc(esz * (size_t)n0);
            double *ximg = (p->kind == O_BOX || p->kind == O_CLAMP) ? (double *)malloc(sizeof(double) * (size_t)n0) : NULL;
            uint32_t *wa = (uint32_t *)calloc(nwords + 1, 4), *wc = (uint32_t *)calloc(nwords + 1, 4);
            uint32_t *wt = (uint32_t *)calloc(nwords + 1, 4);
            int cert[64];
            uint64_t lchk = 0, lv = 0, lf = 0, lcex = UINT64_MAX, lcexu = UINT64_MAX;
            int lbad = 0;
#pragma omp for schedule(dynamic, 8)
            for (int64_t ci = (int64_t)p->begin; ci < (int64_t)p->end; ci++) {
                uint64_t c = (uint64_t)ci;
                if (ximg) orc_decode_box(n->numeric, p, base, n0, b, c, ximg);
                else orc_decode(n->numeric, p, base, n0, b, c, img);
                if (p->restrict_l2 > 0 && !(ximg ? within_restriction_real(n->numeric, base, ximg, n0, p->restrict_l2)
                                                 : within_restriction(n->numeric, base, img, n0, p->restrict_l2)))
                    continue;
                if (forward_d(&dn, img, ximg, tc, h, hn)) lbad = 1;
                int flag;
                int v = property_eval(pr, tc + T - nL, nL, base_cls, V, fl, cov->near_tie, &flag);
                lchk++;
                if (flag) lf++;
                if (v) {
                    lv++;
                    if (c < lcex) lcex = c;
                    if (!flag && c < lcexu) lcexu = c;
                }
                memset(wt, 0, nwords * 4);
                cover_eval(n->sizes, L, tb, tc, cov->n_pairs, cov->lower, dg, dh,
                           fl ? cov->tau : NULL, wt, cert);
                size_t w = 0;
                for (int q = 0; q < cov->n_pairs; q++) {
                    int k = cov->lower[q];
                    size_t wpr = (size_t)(n->sizes[k + 1] + 31) / 32;
                    size_t nw = 2 * (size_t)n->sizes[k] * wpr + 2 * wpr;
                    for (size_t x = w; x < w + nw; x++) {
                        wa[x] |= wt[x];
                        if (!fl || cert[q]) wc[x] |= wt[x];
                    }
                    w += nw;
                }
            }
#pragma omp critical
            {
                checked += lchk; viol += lv; flg += lf;
                if (lcex < cex) cex = lcex;
                if (lcexu < cexu) cexu = lcexu;
                for (size_t x = 0; x < nwords; x++) { res->cov_all[x] |= wa[x]; res->cov_certain[x] |= wc[x]; }
                if (lbad) bad = 1;
            }
            free(tc); free(h); free(hn); free(img); free(ximg); free(wa); free(wc); free(wt);
        }
        res->checked[b] = checked;
        res->violated[b] = viol;
        res->flagged[b] = flg;
        res->first_cex[b] = cex;
        res->first_cex_unflagged[b] = cexu;
        free(tb);
    }
    dnet_free(&dn);
    return bad ? -1 : 0;
}
