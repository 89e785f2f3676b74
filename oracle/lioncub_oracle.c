/* CPU oracle, C restatement, for LARGE parity checks of the Lion Cub step.
 *
 * TEST INFRASTRUCTURE ONLY (like oracle/lioncub_oracle.py): nothing in
 * paper_2411_16462_b200 links or loads it; tests/ use it as the checker at
 * sizes where the numpy oracle needs too much time or host memory
 * (BASELINE.json layouts: GPT-2-small 124M at P = 8, windows of the 1.1B
 * TinyLlama layout and of the 7e9 flat buffer).
 *
 * It restates the reference lioncomm (/root/reference/pkg/src/lioncomm) for
 * all P ranks at once, the same way oracle/lioncub_oracle.py does, and is
 * itself pinned against that numpy oracle and the reference's golden
 * vectors (tests/test_oracle.py::test_c_oracle_*).  Float64 arithmetic in
 * numpy's operand order, compiled with -ffp-contract=off (no FMA) so every
 * product and sum is rounded separately like numpy's:
 *   c      = beta1*m + (1-beta1)*g, masked to 0        optimizer.py:199-201
 *   theta' = theta - eta*(s + wd*theta)                optimizer.py:204
 *   m'     = beta2*m + (1-beta2)*g                     optimizer.py:205
 *   apply_sign (np.sign, zeros -> fill)                quant.py:198-204
 *   L1 quantize: M1 = max|c| * mean(|c|/max|c|) in numpy's pairwise order,
 *     q = clip(round_half_even(qmax/(2 M1) * c), +-qmax)   quant.py:81-104,127-173
 *   compressed_allreduce_1bit: sign tally, apply_sign    collectives.py:252-310
 *   direct_allreduce (binary / offset lanes) -> exact integer sums
 *                                                       collectives.py:179-249
 *   ps_gather_broadcast: f64 sum in rank order (flat) or the binomial tree
 *                                                       collectives.py:96-165
 * fp32 state in, fp32 state out: theta' and m' are float32 of the float64
 * reference values (the CUDA path's 0-ulp contract).
 *
 * Build (by __graft_entry__.build() and the tests, into oracle/_build/):
 *   gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC
 *       oracle/lioncub_oracle.c -o oracle/_build/liblcoracle.so
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { LCO_COMPRESSED1BIT = 0, LCO_DIRECT_SIGNS = 1, LCO_DIRECT_L1 = 2, LCO_PS = 3,
       LCO_PS_EFFICIENT = 4, LCO_PS_SIGNS = 5 };
enum { LCO_OK = 0, LCO_E_ZERO_SIGN = -1, LCO_E_TIE = -2, LCO_E_ARG = -3 };

typedef struct {
  double beta1, one_minus_beta1, beta2, one_minus_beta2, lr, weight_decay;
} lco_hyper;

static inline double lion_c(const lco_hyper* h, float m, float g) {
  return h->beta1 * (double)m + h->one_minus_beta1 * (double)g;
}

/* np.sign with the alternating fill (quant.py:198-204): fill = +1 / -1, or 0
 * for exact-ternary.  -0.0 == 0 takes the fill. */
static inline int sign_fill(double x, int fill) {
  if (x > 0.0) return 1;
  if (x < 0.0) return -1;
  return fill;
}

/* numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src
 * pairwise_sum): < 8 elements sequential; <= 128 elements 8 strided
 * accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus the
 * sequential remainder; larger blocks split at n/2 rounded down to a
 * multiple of 8.  Element i of the summed vector is term(ctx, lo + i). */
typedef double (*term_fn)(const void* ctx, int64_t i);

static double pairwise(term_fn term, const void* ctx, int64_t lo, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += term(ctx, lo + i);
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = term(ctx, lo + k);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; ++k) r[k] += term(ctx, lo + i + k);
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += term(ctx, lo + i);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise(term, ctx, lo, n2) + pairwise(term, ctx, lo + n2, n - n2);
}

typedef struct {
  const float* m;
  const float* g;
  const uint8_t* mask;
  const lco_hyper* h;
  double mx;
} l1_ctx;

static double l1_term(const void* vctx, int64_t i) {
  const l1_ctx* c = (const l1_ctx*)vctx;
  double v = (c->mask && !c->mask[i]) ? 0.0 : lion_c(c->h, c->m[i], c->g[i]);
  return fabs(v) / c->mx;
}

/* lp_mean_norm(c, 1) of one layer (quant.py:81-104) and the quantizer
 * scale qmax / (2 M1) (quant.py:161); scale = 0 marks q == 0 (all-zero c). */
static double l1_scale(const float* m, const float* g, const uint8_t* mask, int64_t n,
                       const lco_hyper* h, int qmax) {
  double mx = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double v = (mask && !mask[i]) ? 0.0 : lion_c(h, m[i], g[i]);
    double a = fabs(v);
    if (a > mx) mx = a;
  }
  if (mx == 0.0 || qmax == 0) return 0.0;
  l1_ctx ctx = {m, g, mask, h, mx};
  double mean = pairwise(l1_term, &ctx, 0, n) / (double)n;
  double M1 = mx * mean;
  if (M1 == 0.0) return 0.0;
  return (double)qmax / (2.0 * M1);
}

static inline int64_t quant_l1(double c, double scale, int qmax) {
  if (scale == 0.0) return 0;
  double r = nearbyint(scale * c); /* round half to even (default FE mode) */
  if (r > qmax) r = qmax;
  if (r < -qmax) r = -qmax;
  return (int64_t)r;
}

/* One Lion Cub step of P ranks on a flat buffer of n elements split into
 * nseg layers (seg_start[0..nseg], sorted-name order).  theta is the shared
 * replica; m[r], g[r] per rank; mask (nullable) per element.  Outputs:
 * theta_out [n], m_out[r] [n] (may alias m[r]), sign_out [n] (nullable),
 * ties [nseg] (nullable).  bits: QuantSpec bits for LCO_DIRECT_L1. */
int lco_step(int P, int64_t n, int nseg, const int64_t* seg_start, const float* theta,
             const float* const* m, const float* const* g, const uint8_t* mask,
             const lco_hyper* h, int algo, int bits, int fill, float* theta_out,
             float* const* m_out, int8_t* sign_out, int64_t* ties) {
  if (P < 1 || P > 64 || n < 0 || nseg < 1 || !seg_start || !theta || !m || !g || !h ||
      !theta_out || !m_out)
    return LCO_E_ARG;
  const int qmax = bits > 1 ? (1 << (bits - 1)) - 1 : 0;
  double* scales = NULL;
  if (algo == LCO_DIRECT_L1) {
    scales = (double*)calloc((size_t)nseg * P, sizeof(double));
    if (!scales) return LCO_E_ARG;
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int s = 0; s < nseg; ++s)
      for (int r = 0; r < P; ++r) {
        const int64_t a = seg_start[s], b = seg_start[s + 1];
        scales[(size_t)s * P + r] =
            b > a ? l1_scale(m[r] + a, g[r] + a, mask ? mask + a : NULL, b - a, h, qmax) : 0.0;
      }
  }
  int err = LCO_OK;
  if (ties)
    for (int s = 0; s < nseg; ++s) ties[s] = 0;
#pragma omp parallel
  {
    int64_t* my_ties = ties ? (int64_t*)calloc((size_t)nseg, sizeof(int64_t)) : NULL;
    int my_err = LCO_OK;
#pragma omp for schedule(static)
    for (int s = 0; s < nseg; ++s) {
      for (int64_t i = seg_start[s]; i < seg_start[s + 1]; ++i) {
        const int keep = mask ? mask[i] != 0 : 1;
        double cs[64];
        for (int r = 0; r < P; ++r) cs[r] = keep ? lion_c(h, m[r][i], g[r][i]) : 0.0;
        int sgn = 0;
        int tie = 0;
        if (algo == LCO_COMPRESSED1BIT) {
          int64_t tally = 0;
          for (int r = 0; r < P; ++r) {
            int sr = sign_fill(cs[r], fill);
            if (sr == 0) my_err = LCO_E_ZERO_SIGN;
            tally += sr;
          }
          tie = tally == 0;
          sgn = sign_fill((double)tally, fill);
          if (sgn == 0) my_err = LCO_E_TIE;
        } else if (algo == LCO_DIRECT_SIGNS || algo == LCO_PS_SIGNS) {
          int64_t sum = 0;
          for (int r = 0; r < P; ++r) {
            int sr = sign_fill(cs[r], fill);
            if (sr == 0 && algo == LCO_DIRECT_SIGNS) my_err = LCO_E_ZERO_SIGN;
            sum += sr;
          }
          tie = sum == 0;
          sgn = sign_fill((double)sum, fill);
        } else if (algo == LCO_DIRECT_L1) {
          int64_t sum = 0;
          for (int r = 0; r < P; ++r) sum += quant_l1(cs[r], scales[(size_t)s * P + r], qmax);
          tie = sum == 0;
          sgn = sign_fill((double)sum, fill);
        } else if (algo == LCO_PS) {
          double tot = cs[0];
          for (int r = 1; r < P; ++r) tot = tot + cs[r];
          tie = tot == 0.0;
          sgn = sign_fill(tot, fill);
        } else if (algo == LCO_PS_EFFICIENT) {
          double acc[64];
          for (int r = 0; r < P; ++r) acc[r] = cs[r];
          for (int mk = 1; mk < P; mk <<= 1)
            for (int r = 0; r + mk < P; r += 2 * mk) acc[r] = acc[r] + acc[r + mk];
          tie = acc[0] == 0.0;
          sgn = sign_fill(acc[0], fill);
        } else {
          my_err = LCO_E_ARG;
        }
        if (my_ties && tie) my_ties[s] += 1;
        if (sign_out) sign_out[i] = (int8_t)sgn;
        const double t = (double)theta[i];
        theta_out[i] = (float)(t - h->lr * ((double)sgn + h->weight_decay * t));
        for (int r = 0; r < P; ++r)
          m_out[r][i] = (float)(h->beta2 * (double)m[r][i] + h->one_minus_beta2 * (double)g[r][i]);
      }
    }
#pragma omp critical
    {
      if (my_ties)
        for (int s = 0; s < nseg; ++s) ties[s] += my_ties[s];
      if (my_err != LCO_OK && err == LCO_OK) err = my_err;
    }
    free(my_ties);
  }
  free(scales);
  return err;
}

/* numpy's pairwise float64 sum of x (test of the restated order). */
static double f64_term(const void* ctx, int64_t i) { return ((const double*)ctx)[i]; }

double lco_pairwise_sum(const double* x, int64_t n) { return pairwise(f64_term, x, 0, n); }

/* Per-layer L1 scale qmax/(2 M1) of one rank (for window checks of the p-bit
 * path: the norm needs the whole layer, the vote only the window). */
int lco_l1_scales(int64_t n, int nseg, const int64_t* seg_start, const float* m, const float* g,
                  const uint8_t* mask, const lco_hyper* h, int bits, double* scales) {
  if (nseg < 1 || !seg_start || !m || !g || !h || !scales || bits < 2) return LCO_E_ARG;
  const int qmax = (1 << (bits - 1)) - 1;
  (void)n;
#pragma omp parallel for schedule(dynamic)
  for (int s = 0; s < nseg; ++s) {
    const int64_t a = seg_start[s], b = seg_start[s + 1];
    scales[s] = b > a ? l1_scale(m + a, g + a, mask ? mask + a : NULL, b - a, h, qmax) : 0.0;
  }
  return LCO_OK;
}
