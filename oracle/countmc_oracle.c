/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see countmc_oracle.h).
 *
 * Plain-C restatement of the reference countmc sweep.  Each function cites
 * the reference file:line it follows (P: = /root/reference/proj/).  Build
 * with -ffp-contract=off: the reference is compiled without FMA
 * (P:CMakeLists.txt:7-9,30), and expression order below follows C++
 * left-to-right evaluation of the cited lines exactly.
 */
#include "countmc_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ RNG */

/* Philox4x64-10 round constants and Weyl key bumps, P:src/rng.cpp:10-13. */
static const uint64_t kMul0 = 0xD2E7470EE14C6C93ull;
static const uint64_t kMul1 = 0xCA5A826395121157ull;
static const uint64_t kWeyl0 = 0x9E3779B97F4A7C15ull;
static const uint64_t kWeyl1 = 0xBB67AE8584CAA73Bull;

/* P:src/rng.cpp:15-44 */
void orc_philox4x64(const uint64_t ctr_in[4], const uint64_t key_in[2],
                    uint64_t out[4]) {
  uint64_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
  uint64_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += kWeyl0;
      k1 += kWeyl1;
    }
    unsigned __int128 p0 = (unsigned __int128)kMul0 * c[0];
    unsigned __int128 p1 = (unsigned __int128)kMul1 * c[2];
    uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    uint64_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
    c[0] = n0;
    c[1] = n1;
    c[2] = n2;
    c[3] = n3;
  }
  out[0] = c[0];
  out[1] = c[1];
  out[2] = c[2];
  out[3] = c[3];
}

/* RngStream ctor, key=(seed, chain), ctr=(iteration, site, 0, 0),
 * P:include/countmc/rng.hpp:23-25. */
void orc_stream_init(orc_stream* s, uint64_t seed, uint64_t chain,
                     uint64_t iteration, uint64_t site) {
  s->ctr[0] = iteration;
  s->ctr[1] = site;
  s->ctr[2] = 0;
  s->ctr[3] = 0;
  s->key[0] = seed;
  s->key[1] = chain;
  s->pos = 4;
}

/* operator() and refill, P:include/countmc/rng.hpp:32-35,52-56. */
uint64_t orc_next(orc_stream* s) {
  if (s->pos == 4) {
    orc_philox4x64(s->ctr, s->key, s->buf);
    ++s->ctr[2];
    s->pos = 0;
  }
  return s->buf[s->pos++];
}

/* P:include/countmc/rng.hpp:38-40 */
double orc_u01(orc_stream* s) {
  return ((double)(orc_next(s) >> 11) + 0.5) * 0x1.0p-53;
}

/* P:src/rng.cpp:76-83 */
uint64_t orc_uniform_int(orc_stream* s, uint64_t n) {
  const uint64_t reject_below = (0u - n) % n;
  for (;;) {
    const uint64_t x = orc_next(s);
    if (x >= reject_below) return x % n;
  }
}

/* P:src/rng.cpp:46 */
double orc_normal(orc_stream* s) { return orc_normal_quantile(orc_u01(s)); }

/* Marsaglia-Tsang with the shape<1 boost and the 1e-300 floor,
 * P:src/rng.cpp:48-74. */
double orc_gamma(orc_stream* s, double shape, double rate) {
  if (!(shape > 0.0) || !(rate > 0.0)) return NAN;
  double boost = 1.0;
  if (shape < 1.0) {
    boost = pow(orc_u01(s), 1.0 / shape);
    shape += 1.0;
  }
  const double d = shape - 1.0 / 3.0;
  const double c = 1.0 / (3.0 * sqrt(d));
  for (;;) {
    double x, v;
    do {
      x = orc_normal(s);
      v = 1.0 + c * x;
    } while (v <= 0.0);
    v = v * v * v;
    const double u = orc_u01(s);
    const double x2 = x * x;
    if (u < 1.0 - 0.0331 * x2 * x2 ||
        log(u) < 0.5 * x2 + d * (1.0 - v + log(v))) {
      double draw = boost * d * v / rate;
      if (draw < 1e-300) draw = 1e-300;
      return draw;
    }
  }
}

/* Wichura AS241 PPND16, three regions, P:src/rng.cpp:88-146.  The
 * coefficients are the published AS241 constants. */
static double orc_ratio(const double* num, const double* den, double r) {
  double n = num[7], d = den[7];
  for (int i = 6; i >= 0; --i) {
    n = n * r + num[i];
    d = d * r + den[i];
  }
  return n / d;
}

double orc_normal_quantile(double p) {
  static const double a[8] = {
      3.3871328727963666080e+00, 1.3314166789178437745e+02,
      1.9715909503065514427e+03, 1.3731693765509461125e+04,
      4.5921953931549871457e+04, 6.7265770927008700853e+04,
      3.3430575583588128105e+04, 2.5090809287301226727e+03};
  static const double b[8] = {
      1.0, 4.2313330701600911252e+01, 6.8718700749205790830e+02,
      5.3941960214247511077e+03, 2.1213794301586595867e+04,
      3.9307895800092710610e+04, 2.8729085735721942674e+04,
      5.2264952788528545610e+03};
  static const double c[8] = {
      1.42343711074968357734e+00, 4.63033784615654529590e+00,
      5.76949722146069140550e+00, 3.64784832476320460504e+00,
      1.27045825245236838258e+00, 2.41780725177450611770e-01,
      2.27238449892691845833e-02, 7.74545014278341407640e-04};
  static const double dd[8] = {
      1.0, 2.05319162663775882187e+00, 1.67638483018380384940e+00,
      6.89767334985100004550e-01, 1.48103976427480074590e-01,
      1.51986665636164571966e-02, 5.47593808499534494600e-04,
      1.05075007164441684324e-09};
  static const double e[8] = {
      6.65790464350110377720e+00, 5.46378491116411436990e+00,
      1.78482653991729133580e+00, 2.96560571828504891230e-01,
      2.65321895265761230930e-02, 1.24266094738807843860e-03,
      2.71155556874348757815e-05, 2.01033439929228813265e-07};
  static const double f[8] = {
      1.0, 5.99832206555887937690e-01, 1.36929880922735805310e-01,
      1.48753612908506148525e-02, 7.86869131145613259100e-04,
      1.84631831751005468180e-05, 1.42151175831644588870e-07,
      2.04426310338993978564e-15};
  if (!(p > 0.0) || !(p < 1.0)) return NAN;
  const double q = p - 0.5;
  if (fabs(q) <= 0.425) {
    const double r = 0.180625 - q * q;
    return q * orc_ratio(a, b, r);
  }
  double r = (q < 0.0) ? p : 1.0 - p;
  r = sqrt(-log(r));
  double value;
  if (r <= 5.0)
    value = orc_ratio(c, dd, r - 1.6);
  else
    value = orc_ratio(e, f, r - 5.0);
  return (q < 0.0) ? -value : value;
}

void orc_stream_u01(uint64_t seed, uint64_t chain, uint64_t it, uint64_t site,
                    long n, double* out) {
  orc_stream s;
  orc_stream_init(&s, seed, chain, it, site);
  for (long i = 0; i < n; ++i) out[i] = orc_u01(&s);
}

/* ---------------------------------------------------------------- model */

static const double kExpClamp = 700.0; /* P:include/countmc/model.hpp:14 */

/* P:src/model.cpp:13-19 */
double orc_clamped_exp(double x, uint64_t* clamps) {
  if (x > kExpClamp) {
    if (clamps) ++*clamps;
    x = kExpClamp;
  }
  return exp(x);
}

/* P:src/model.cpp:70-74 */
double orc_log_fc_epsilon(long long y, double h, double eta, double gamma,
                          double eps, uint64_t* clamps) {
  return (double)y * eps - orc_clamped_exp(h + eta + eps, clamps) -
         eps * eps / (2.0 * gamma);
}

/* P:src/model.cpp:76-82 */
void orc_gamma_fc_params(double nu, double tau, const double* eps_row,
                         long N, double* shape, double* scale) {
  double ss = 0.0;
  for (long n = 0; n < N; ++n) ss += eps_row[n] * eps_row[n];
  *shape = (nu + (double)N) / 2.0;
  *scale = (nu * tau + ss) / 2.0;
}

/* P:src/model.cpp:84-87 */
double orc_log_invgamma(double x, double shape, double scale) {
  if (!(x > 0.0)) return -INFINITY;
  return -(shape + 1.0) * log(x) - scale / x;
}

/* P:src/model.cpp:89-92 */
double orc_log_gamma_rate(double x, double shape, double rate) {
  if (!(x > 0.0)) return -INFINITY;
  return (shape - 1.0) * log(x) - rate * x;
}

/* P:src/model.cpp:94-100 */
double orc_log_fc_nu(double nu, long G, double tau, double sum_log_gamma,
                     double sum_inv_gamma, double d) {
  if (!(nu > 0.0) || !(nu < d)) return -INFINITY;
  const double Gd = (double)G;
  return -Gd * lgamma(nu / 2.0) + (Gd * nu / 2.0) * log(nu * tau / 2.0) -
         (nu / 2.0) * (sum_log_gamma + tau * sum_inv_gamma);
}

/* P:src/model.cpp:102-105 */
void orc_tau_fc_params(double a, double b, long G, double nu,
                       double sum_inv_gamma, double* shape, double* rate) {
  *shape = a + (double)G * nu / 2.0;
  *rate = b + (nu / 2.0) * sum_inv_gamma;
}

/* P:src/model.cpp:124-129 */
void orc_theta_fc_params(double sum_beta, long G, double sigma, double c,
                         double* mean, double* sd) {
  const double v = 1.0 / (1.0 / (c * c) + (double)G / (sigma * sigma));
  *mean = v * sum_beta / (sigma * sigma);
  *sd = sqrt(v);
}

/* P:src/model.cpp:131-136 */
double orc_log_fc_sigma(double sigma, long G, double ss, double s_bound) {
  if (!(sigma > 0.0) || !(sigma < s_bound)) return -INFINITY;
  return -(double)G * log(sigma) - ss / (2.0 * sigma * sigma);
}

/* xi full conditional (extension, no reference: parity unpinned).  With
 * q = (beta - theta)^2 / (2 sigma^2) and beta ~ N(theta, sigma^2 xi):
 *   laplace   xi ~ Exp(rate 1/2):        -log(xi)/2 - q/xi - xi/2
 *   t(k)      xi ~ IG(k/2, k/2):         -(k/2 + 3/2) log(xi) - (q + k/2)/xi
 *   horseshoe sqrt(xi) ~ Cauchy+(0,1):   -log(xi) - q/xi - log1p(xi),
 *             evaluated as -log(xi (1 + xi)) - q/xi (one log) below 1e150
 * and -inf for xi <= 0. */
double orc_log_fc_xi(int prior, double xi, double q, double k) {
  if (!(xi > 0.0)) return -INFINITY;
  switch (prior) {
    case CMC_PRIOR_LAPLACE:
      return -0.5 * log(xi) - q / xi - 0.5 * xi;
    case CMC_PRIOR_T:
      return -(0.5 * k + 1.5) * log(xi) - (q + 0.5 * k) / xi;
    case CMC_PRIOR_HORSESHOE:
      return xi < 1e150 ? -log(xi * (1.0 + xi)) - q / xi : -log(xi) - q / xi - log1p(xi);
    default:
      return 0.0;
  }
}

/* ---------------------------------------------------------------- slice */

/* P:include/countmc/slice.hpp:27-35 */
void orc_tune_update(double* w, double* w_aux, long m, double delta,
                     const orc_slice_cfg* cfg) {
  const double md = (double)m;
  *w_aux += md * delta;
  if (m > cfg->tune_cutoff) {
    const double nw = *w_aux / (0.5 * md * (md + 1.0));
    if (nw >= 1e-12) *w = nw;
  }
}

/* Stepping out + shrinkage, draw order as P:include/countmc/slice.hpp:42-75. */
double orc_slice_step(orc_logf f, void* ctx, double x0, double* w,
                      double* w_aux, const orc_slice_cfg* cfg, long m,
                      orc_stream* rng, int* stalled) {
  const double fx0 = f(ctx, x0);
  const double logu = fx0 + log(orc_u01(rng));
  const double wv = *w;
  double lo = x0 - wv * orc_u01(rng);
  double hi = lo + wv;
  uint64_t kl = orc_uniform_int(rng, (uint64_t)cfg->max_step_out + 1);
  uint64_t kr = (uint64_t)cfg->max_step_out - kl;
  while (kl > 0 && logu < f(ctx, lo)) {
    lo -= wv;
    --kl;
  }
  while (kr > 0 && logu < f(ctx, hi)) {
    hi += wv;
    --kr;
  }
  for (int it = 0; it < cfg->max_shrink; ++it) {
    const double x1 = lo + (hi - lo) * orc_u01(rng);
    if (f(ctx, x1) > logu) {
      if (m <= cfg->burnin) orc_tune_update(w, w_aux, m, fabs(x1 - x0), cfg);
      return x1;
    }
    if (x1 > x0)
      hi = x1;
    else
      lo = x1;
  }
  *stalled = 1;
  return x0;
}

static double d_normal(void* c, double x) {
  (void)c;
  return -x * x / 2.0;
}
static double d_gamma32(void* c, double x) {
  (void)c;
  return x > 0.0 ? 2.0 * log(x) - 2.0 * x : -INFINITY;
}
static double d_invgamma23(void* c, double x) {
  (void)c;
  return x > 0.0 ? -3.0 * log(x) - 3.0 / x : -INFINITY;
}
static double d_box(void* c, double x) {
  (void)c;
  return (x > 0.0 && x < 1.0) ? 0.0 : -INFINITY;
}
/* xi conditionals at q = 0.7 (t: k = 3, i.e. IG(2, 2.2)) */
static double d_xi_t(void* c, double x) {
  (void)c;
  return orc_log_fc_xi(CMC_PRIOR_T, x, 0.7, 3.0);
}
static double d_xi_laplace(void* c, double x) {
  (void)c;
  return orc_log_fc_xi(CMC_PRIOR_LAPLACE, x, 0.7, 0.0);
}
static double d_xi_horseshoe(void* c, double x) {
  (void)c;
  return orc_log_fc_xi(CMC_PRIOR_HORSESHOE, x, 0.7, 0.0);
}

/* run_chain helper of P:tests/test_slice.cpp:21-39. */
int orc_slice_chain(int density, double x0, long n, long burnin,
                    double w_init, uint64_t seed, double* out) {
  orc_logf f = density == 0   ? d_normal
               : density == 1 ? d_gamma32
               : density == 2 ? d_invgamma23
               : density == 3 ? d_box
               : density == 4 ? d_xi_t
               : density == 5 ? d_xi_laplace
                              : d_xi_horseshoe;
  orc_slice_cfg cfg = {100, burnin, burnin / 10, w_init, 1000};
  double w = w_init, waux = 0.0, x = x0;
  long k = 0;
  for (long m = 1; m <= burnin + n; ++m) {
    orc_stream rng;
    orc_stream_init(&rng, seed, 0, (uint64_t)m, 0);
    int st = 0;
    x = orc_slice_step(f, NULL, x, &w, &waux, &cfg, m, &rng, &st);
    if (st) return 2;
    if (m > burnin) out[k++] = x;
  }
  return 0;
}

/* ----------------------------------------------------------- reductions */

/* P:src/parallel.cpp:81-86 */
double orc_pairwise_sum(const double* x, size_t n) {
  if (n == 0) return 0.0;
  if (n == 1) return x[0];
  const size_t mid = n / 2;
  return orc_pairwise_sum(x, mid) + orc_pairwise_sum(x + mid, n - mid);
}

/* det_transform_sum with kReduceBlock = 1024, P:include/countmc/parallel.hpp:57-84 */
double orc_det_sum(const double* x, long n) {
  if (n <= 0) return 0.0;
  const long nb = (n + 1023) / 1024;
  double* sums = (double*)malloc(sizeof(double) * (size_t)nb);
  for (long b = 0; b < nb; ++b) {
    const long lo = b * 1024;
    const long hi = (lo + 1024 < n) ? lo + 1024 : n;
    double s = 0.0;
    for (long i = lo; i < hi; ++i) s += x[i];
    sums[b] = s;
  }
  const double r = orc_pairwise_sum(sums, (size_t)nb);
  free(sums);
  return r;
}

/* ------------------------------------------------------------ streaming */

/* Kahan add, P:include/countmc/streaming.hpp:29-34 */
static void kahan(double* sum, double* comp, double term) {
  const double y = term - *comp;
  const double t = *sum + y;
  *comp = (t - *sum) - y;
  *sum = t;
}

/* MomentAccumulator::update, P:include/countmc/streaming.hpp:17-22 */
void orc_moments_update(orc_moments* a, double value) {
  ++a->count;
  const double m = (double)a->count;
  kahan(&a->mean, &a->mean_c, (value - a->mean) / m);
  kahan(&a->meansq, &a->meansq_c, (value * value - a->meansq) / m);
}

void orc_moments_stream(const double* v, long n, double* mean,
                        double* meansq) {
  orc_moments a = {0, 0.0, 0.0, 0.0, 0.0};
  for (long i = 0; i < n; ++i) orc_moments_update(&a, v[i]);
  *mean = a.mean;
  *meansq = a.meansq;
}

/* P:src/streaming.cpp:110-112 */
double orc_disjunction_combine(double p1, double p2, double p12) {
  double v = p1 + p2 - p12;
  if (v < 0.0) v = 0.0;
  if (v > 1.0) v = 1.0;
  return v;
}

/* --------------------------------------------------------------- engine */

/* Draw-site families, P:include/countmc/engine.hpp:42-49 */
enum { kEps = 1, kGamma = 2, kNu = 3, kTau = 4, kBeta = 5, kTheta = 6,
       kSigma = 7, kSaveSel = 8, kXi = 11 /* extension: xi priors */ };
static uint64_t site_id(uint64_t fam, uint64_t flat) {
  return (fam << 56) | flat;
}

typedef struct orc_group {
  double value;
  long n_idx;
  long* idx;
} orc_group;

typedef struct orc_contrast {
  int n_terms;
  int* n_coefs;
  double* threshold;
  int** family;
  int** index;
  double** coef;
  int per_gene;
} orc_contrast;

struct orc_engine {
  long G, N, L;
  long long* y; /* G x N */
  double* X;    /* N x L */
  double* h;
  double a, b, d;
  double* c;
  double* s;
  cmc_run_config cfg;
  orc_slice_cfg scfg;
  double* A; /* G x L */
  long* n_groups;
  orc_group** groups;
  long n_saved;
  long* saved;
  int n_contrasts;
  orc_contrast* contrasts;
  /* xi-augmented beta priors (extension, no reference: parity unpinned) */
  int xi_any;
  int* prior; /* L: CMC_PRIOR_* */
  double t_df;
};

static void set_err(cmc_error* err, int code, const char* msg) {
  if (!err) return;
  memset(err, 0, sizeof(*err));
  err->code = code;
  err->index1 = err->index2 = -1;
  snprintf(err->msg, sizeof(err->msg), "%s", msg);
}

/* SamplerStallError formatting, P:src/errors.cpp:8-16, annotated as the
 * engine rethrows it (P:src/engine.cpp:196-198 etc.). */
static void set_stall(cmc_error* err, const char* step, long i1, long i2,
                      double x0, double w, long m) {
  if (!err) return;
  memset(err, 0, sizeof(*err));
  err->code = CMC_ERR_STALL;
  snprintf(err->step, sizeof(err->step), "%s", step);
  err->index1 = i1;
  err->index2 = i2;
  err->x0 = x0;
  err->width = w;
  err->iteration = m;
  snprintf(err->msg, sizeof(err->msg),
           "slice sampler stalled: step=%s index=(%ld,%ld) x0=%.17g "
           "width=%.17g iteration=%ld",
           step[0] ? step : "?", i1, i2, x0, w, m);
}

static long matrix_rank(const double* Xin, long n, long m, double tol) {
  double* A = (double*)malloc(sizeof(double) * (size_t)(n * m));
  memcpy(A, Xin, sizeof(double) * (size_t)(n * m));
  double maxabs = 0.0;
  for (long i = 0; i < n * m; ++i)
    if (fabs(A[i]) > maxabs) maxabs = fabs(A[i]);
  if (maxabs == 0.0) {
    free(A);
    return 0;
  }
  const double thresh = tol * maxabs;
  long rank = 0;
  for (long col = 0; col < m && rank < n; ++col) {
    long pivot = rank;
    for (long r = rank + 1; r < n; ++r)
      if (fabs(A[r * m + col]) > fabs(A[pivot * m + col])) pivot = r;
    if (fabs(A[pivot * m + col]) <= thresh) continue;
    if (pivot != rank)
      for (long cc = 0; cc < m; ++cc) {
        double t = A[pivot * m + cc];
        A[pivot * m + cc] = A[rank * m + cc];
        A[rank * m + cc] = t;
      }
    for (long r = rank + 1; r < n; ++r) {
      const double fct = A[r * m + col] / A[rank * m + col];
      for (long cc = col; cc < m; ++cc) A[r * m + cc] -= fct * A[rank * m + cc];
    }
    ++rank;
  }
  free(A);
  return rank;
}

static int cmp_long(const void* a, const void* b) {
  long x = *(const long*)a, y = *(const long*)b;
  return (x > y) - (x < y);
}

/* GibbsEngine ctor, P:src/engine.cpp:42-91 (+ RunConfig::resolve :25-40,
 * validation P:src/types.cpp:18-69, ContrastSpec::finalize
 * P:src/streaming.cpp:76-88). */
int orc_engine_create(const cmc_problem* p, const cmc_run_config* cfg_in,
                      const cmc_contrast_set* cs, orc_engine** out,
                      cmc_error* err) {
  *out = NULL;
  if (p->G < 1 || p->N < 1) {
    set_err(err, CMC_ERR_CONFIG,
            "count matrix must have at least one gene and one sample");
    return CMC_ERR_CONFIG;
  }
  if (p->L < 1) {
    set_err(err, CMC_ERR_CONFIG,
            "model matrix must have at least one row and one column");
    return CMC_ERR_CONFIG;
  }
  for (long i = 0; i < p->G * p->N; ++i)
    if (p->counts[i] < 0) {
      set_err(err, CMC_ERR_CONFIG, "negative count");
      return CMC_ERR_CONFIG;
    }
  for (long i = 0; i < p->N; ++i)
    if (!isfinite(p->h[i])) {
      set_err(err, CMC_ERR_CONFIG, "offsets must be finite");
      return CMC_ERR_CONFIG;
    }
  for (long i = 0; i < p->N * p->L; ++i)
    if (!isfinite(p->X[i])) {
      set_err(err, CMC_ERR_CONFIG, "model matrix entries must be finite");
      return CMC_ERR_CONFIG;
    }
  if (matrix_rank(p->X, p->N, p->L, 1e-10) < p->L) {
    set_err(err, CMC_ERR_CONFIG, "model matrix does not have full column rank");
    return CMC_ERR_CONFIG;
  }
  if (!(p->a > 0.0) || !(p->b > 0.0) || !(p->d > 0.0)) {
    set_err(err, CMC_ERR_CONFIG, "prior constants a, b, d must be strictly positive");
    return CMC_ERR_CONFIG;
  }
  for (long l = 0; l < p->L; ++l)
    if (!(p->c[l] > 0.0) || !(p->s[l] > 0.0)) {
      set_err(err, CMC_ERR_CONFIG, "prior entries c, s must be strictly positive");
      return CMC_ERR_CONFIG;
    }
  if (p->beta_prior)
    for (long l = 0; l < p->L; ++l) {
      if (p->beta_prior[l] < CMC_PRIOR_NORMAL || p->beta_prior[l] > CMC_PRIOR_HORSESHOE) {
        set_err(err, CMC_ERR_CONFIG, "beta prior must be normal, laplace, t or horseshoe");
        return CMC_ERR_CONFIG;
      }
      if (p->beta_prior[l] == CMC_PRIOR_T && !(p->t_df > 0.0)) {
        set_err(err, CMC_ERR_CONFIG, "t prior needs positive degrees of freedom");
        return CMC_ERR_CONFIG;
      }
    }
  cmc_run_config cfg = *cfg_in;
  const char* bad = NULL;
  if (cfg.chains < 1) bad = "chains must be >= 1";
  else if (cfg.iterations < 1) bad = "iterations must be >= 1";
  else if (cfg.burnin < 1) bad = "burnin must be >= 1";
  else if (cfg.thin < 1) bad = "thin must be >= 1";
  else if (cfg.workers < 1) bad = "workers must be >= 1";
  else if (cfg.save_genes < 0) bad = "save_genes must be >= 0";
  else if (cfg.max_step_out < 1) bad = "max_step_out must be >= 1";
  if (!bad) {
    if (cfg.tune_cutoff < 0)
      cfg.tune_cutoff = cfg.burnin / 10 < 500 ? cfg.burnin / 10 : 500;
    if (cfg.tune_cutoff >= cfg.burnin)
      bad = "tune_cutoff must be less than burnin (M_C < M_B)";
    else if (!(cfg.w_init > 0.0)) bad = "w_init must be positive";
    else if (cfg.max_shrink < 1) bad = "max_shrink must be >= 1";
  }
  if (bad) {
    set_err(err, CMC_ERR_CONFIG, bad);
    return CMC_ERR_CONFIG;
  }

  orc_engine* e = (orc_engine*)calloc(1, sizeof(orc_engine));
  const long G = p->G, N = p->N, L = p->L;
  e->G = G;
  e->N = N;
  e->L = L;
  e->y = (long long*)malloc(sizeof(long long) * (size_t)(G * N));
  memcpy(e->y, p->counts, sizeof(long long) * (size_t)(G * N));
  e->X = (double*)malloc(sizeof(double) * (size_t)(N * L));
  memcpy(e->X, p->X, sizeof(double) * (size_t)(N * L));
  e->h = (double*)malloc(sizeof(double) * (size_t)N);
  memcpy(e->h, p->h, sizeof(double) * (size_t)N);
  e->a = p->a;
  e->b = p->b;
  e->d = p->d;
  e->c = (double*)malloc(sizeof(double) * (size_t)L);
  e->s = (double*)malloc(sizeof(double) * (size_t)L);
  memcpy(e->c, p->c, sizeof(double) * (size_t)L);
  memcpy(e->s, p->s, sizeof(double) * (size_t)L);
  e->prior = (int*)calloc((size_t)L, sizeof(int));
  if (p->beta_prior) memcpy(e->prior, p->beta_prior, sizeof(int) * (size_t)L);
  for (long l = 0; l < L; ++l) e->xi_any |= e->prior[l] != CMC_PRIOR_NORMAL;
  e->t_df = p->t_df;
  e->cfg = cfg;
  e->scfg.max_step_out = cfg.max_step_out;
  e->scfg.burnin = cfg.burnin;
  e->scfg.tune_cutoff = cfg.tune_cutoff;
  e->scfg.w_init = cfg.w_init;
  e->scfg.max_shrink = cfg.max_shrink;

  /* A_gl = sum_n y_gn X_nl, P:src/engine.cpp:55-60 */
  e->A = (double*)calloc((size_t)(G * L), sizeof(double));
  for (long g = 0; g < G; ++g)
    for (long n = 0; n < N; ++n) {
      const double yv = (double)e->y[g * N + n];
      for (long l = 0; l < L; ++l) e->A[g * L + l] += yv * e->X[n * L + l];
    }

  /* column groups, P:src/engine.cpp:62-75 */
  e->n_groups = (long*)calloc((size_t)L, sizeof(long));
  e->groups = (orc_group**)calloc((size_t)L, sizeof(orc_group*));
  for (long l = 0; l < L; ++l) {
    e->groups[l] = (orc_group*)calloc((size_t)N, sizeof(orc_group));
    for (long n = 0; n < N; ++n) {
      const double v = e->X[n * L + l];
      if (v == 0.0) continue;
      long j = 0;
      for (; j < e->n_groups[l]; ++j)
        if (e->groups[l][j].value == v) break;
      if (j == e->n_groups[l]) {
        e->groups[l][j].value = v;
        e->groups[l][j].idx = (long*)malloc(sizeof(long) * (size_t)N);
        e->groups[l][j].n_idx = 0;
        ++e->n_groups[l];
      }
      e->groups[l][j].idx[e->groups[l][j].n_idx++] = n;
    }
  }

  /* saved genes: partial Fisher-Yates then sort, P:src/engine.cpp:77-90 */
  const long k = cfg.save_genes < G ? cfg.save_genes : G;
  e->n_saved = k;
  e->saved = (long*)malloc(sizeof(long) * (size_t)(k > 0 ? k : 1));
  if (k > 0) {
    long* idx = (long*)malloc(sizeof(long) * (size_t)G);
    for (long i = 0; i < G; ++i) idx[i] = i;
    orc_stream sel;
    orc_stream_init(&sel, cfg.seed, 0, 0, site_id(kSaveSel, 0));
    for (long i = 0; i < k; ++i) {
      const long j = i + (long)orc_uniform_int(&sel, (uint64_t)(G - i));
      long t = idx[i];
      idx[i] = idx[j];
      idx[j] = t;
    }
    memcpy(e->saved, idx, sizeof(long) * (size_t)k);
    qsort(e->saved, (size_t)k, sizeof(long), cmp_long);
    free(idx);
  }

  /* contrasts */
  if (cs && cs->n_contrasts > 0) {
    e->n_contrasts = cs->n_contrasts;
    e->contrasts = (orc_contrast*)calloc((size_t)cs->n_contrasts, sizeof(orc_contrast));
    int t = 0, q = 0;
    for (int ci = 0; ci < cs->n_contrasts; ++ci) {
      orc_contrast* oc = &e->contrasts[ci];
      oc->n_terms = cs->n_terms[ci];
      if (oc->n_terms < 1) {
        set_err(err, CMC_ERR_CONFIG, "contrast has no terms");
        orc_engine_destroy(e);
        return CMC_ERR_CONFIG;
      }
      oc->n_coefs = (int*)calloc((size_t)oc->n_terms, sizeof(int));
      oc->threshold = (double*)calloc((size_t)oc->n_terms, sizeof(double));
      oc->family = (int**)calloc((size_t)oc->n_terms, sizeof(int*));
      oc->index = (int**)calloc((size_t)oc->n_terms, sizeof(int*));
      oc->coef = (double**)calloc((size_t)oc->n_terms, sizeof(double*));
      for (int ti = 0; ti < oc->n_terms; ++ti, ++t) {
        const int nc = cs->n_coefs[t];
        if (nc < 1) {
          set_err(err, CMC_ERR_CONFIG, "contrast has a term with no coefficients");
          orc_engine_destroy(e);
          return CMC_ERR_CONFIG;
        }
        oc->n_coefs[ti] = nc;
        oc->threshold[ti] = cs->threshold[t];
        oc->family[ti] = (int*)malloc(sizeof(int) * (size_t)nc);
        oc->index[ti] = (int*)malloc(sizeof(int) * (size_t)nc);
        oc->coef[ti] = (double*)malloc(sizeof(double) * (size_t)nc);
        for (int k2 = 0; k2 < nc; ++k2, ++q) {
          oc->family[ti][k2] = cs->family[q];
          oc->index[ti][k2] = cs->index[q];
          oc->coef[ti][k2] = cs->coef[q];
          if (cs->family[q] == CMC_FAM_BETA_COL || cs->family[q] == CMC_FAM_GAMMA)
            oc->per_gene = 1;
        }
      }
    }
  }
  *out = e;
  return CMC_OK;
}

void orc_engine_destroy(orc_engine* e) {
  if (!e) return;
  free(e->y);
  free(e->X);
  free(e->h);
  free(e->c);
  free(e->s);
  free(e->prior);
  free(e->A);
  if (e->groups) {
    for (long l = 0; l < e->L; ++l) {
      for (long j = 0; j < e->n_groups[l]; ++j) free(e->groups[l][j].idx);
      free(e->groups[l]);
    }
    free(e->groups);
  }
  free(e->n_groups);
  free(e->saved);
  for (int ci = 0; ci < e->n_contrasts; ++ci) {
    orc_contrast* oc = &e->contrasts[ci];
    for (int ti = 0; ti < oc->n_terms; ++ti) {
      if (oc->family) free(oc->family[ti]);
      if (oc->index) free(oc->index[ti]);
      if (oc->coef) free(oc->coef[ti]);
    }
    free(oc->n_coefs);
    free(oc->threshold);
    free(oc->family);
    free(oc->index);
    free(oc->coef);
  }
  free(e->contrasts);
  free(e);
}

int orc_engine_config(const orc_engine* e, cmc_run_config* out) {
  *out = e->cfg;
  return CMC_OK;
}
long orc_engine_n_saved(const orc_engine* e) { return e->n_saved; }
int orc_engine_saved_genes(const orc_engine* e, long* out) {
  for (long i = 0; i < e->n_saved; ++i) out[i] = e->saved[i];
  return CMC_OK;
}

/* Packed-state offsets (include/countmc_b200.h). */
#define ST_EPS(e) 0
#define ST_GAMMA(e) ((e)->G * (e)->N)
#define ST_BETA(e) (ST_GAMMA(e) + (e)->G)
#define ST_THETA(e) (ST_BETA(e) + (e)->G * (e)->L)
#define ST_SIGMA(e) (ST_THETA(e) + (e)->L)
#define ST_NU(e) (ST_SIGMA(e) + (e)->L)
#define ST_TAU(e) (ST_NU(e) + 1)
#define TU_EPS(e) 0
#define TU_GAMMA(e) ((e)->G * (e)->N)
#define TU_BETA(e) (TU_GAMMA(e) + (e)->G)
#define TU_SIGMA(e) (TU_BETA(e) + (e)->G * (e)->L)
#define TU_NU(e) (TU_SIGMA(e) + (e)->L)
#define TU_TAU(e) (TU_NU(e) + 1)
#define ST_XI(e) (ST_TAU(e) + 1)
#define TU_XI(e) (TU_TAU(e) + 1)

static double std_max(double a, double b) { return (a < b) ? b : a; }
static double std_min(double a, double b) { return (b < a) ? b : a; }

/* P:src/engine.cpp:98-142 */
int orc_initial_state(const orc_engine* e, long chain, double* st) {
  const long G = e->G, N = e->N, L = e->L;
  double* eps = st + ST_EPS(e);
  double* gam = st + ST_GAMMA(e);
  double* beta = st + ST_BETA(e);
  double* theta = st + ST_THETA(e);
  double* sigma = st + ST_SIGMA(e);
  for (long i = 0; i < G * N; ++i) eps[i] = 0.0;
  for (long g = 0; g < G; ++g) gam[g] = 1.0;
  for (long i = 0; i < G * L; ++i) beta[i] = 0.0;
  for (long l = 0; l < L; ++l) {
    theta[l] = 0.0;
    sigma[l] = 1.0;
  }
  st[ST_NU(e)] = 2.0;
  st[ST_TAU(e)] = 1.0;
  if (e->xi_any)
    for (long i = 0; i < G * L; ++i) st[ST_XI(e) + i] = 1.0;

  double hbar = 0.0;
  for (long n = 0; n < N; ++n) hbar += e->h[n];
  hbar /= (double)N;
  for (long g = 0; g < G; ++g) {
    double mean = 0.0;
    for (long n = 0; n < N; ++n) mean += (double)e->y[g * N + n];
    mean /= (double)N;
    beta[g * L + 0] = log(mean + 1.0) - hbar;
  }
  double tbar = 0.0;
  for (long g = 0; g < G; ++g) tbar += beta[g * L + 0];
  theta[0] = tbar / (double)G;

  if (chain > 0) {
    const uint64_t seed = e->cfg.seed, ch = (uint64_t)chain;
#define Z(fam, flat)                                               \
  (__extension__({                                                 \
    orc_stream zs_;                                                \
    orc_stream_init(&zs_, seed, ch, 0, site_id((fam), (flat)));    \
    0.5 * orc_normal(&zs_);                                        \
  }))
    for (long g = 0; g < G; ++g) {
      for (long n = 0; n < N; ++n) eps[g * N + n] += Z(kEps, (uint64_t)(g * N + n));
      gam[g] = std_max(1e-3, gam[g] + Z(kGamma, (uint64_t)g));
      for (long l = 0; l < L; ++l) beta[g * L + l] += Z(kBeta, (uint64_t)(g * L + l));
    }
    for (long l = 0; l < L; ++l) {
      theta[l] += Z(kTheta, (uint64_t)l);
      const double sv = e->s[l];
      sigma[l] = std_min(std_max(sigma[l] + Z(kSigma, (uint64_t)l), 1e-6 * sv),
                         (1.0 - 1e-6) * sv);
    }
    st[ST_NU(e)] = std_min(std_max(st[ST_NU(e)] + Z(kNu, 0), 1e-6 * e->d),
                           (1.0 - 1e-6) * e->d);
    st[ST_TAU(e)] = std_max(1e-3, st[ST_TAU(e)] + Z(kTau, 0));
#undef Z
  }
  return CMC_OK;
}

/* log-density closures */
typedef struct {
  long long y;
  double h, eta, gamma;
  uint64_t* clamps;
} eps_ctx;
static double f_eps(void* c, double x) {
  eps_ctx* k = (eps_ctx*)c;
  return orc_log_fc_epsilon(k->y, k->h, k->eta, k->gamma, x, k->clamps);
}
typedef struct {
  double shape, scale;
} ig_ctx;
static double f_ig(void* c, double x) {
  ig_ctx* k = (ig_ctx*)c;
  return orc_log_invgamma(x, k->shape, k->scale);
}
static double f_gr(void* c, double x) {
  ig_ctx* k = (ig_ctx*)c;
  return orc_log_gamma_rate(x, k->shape, k->scale);
}
typedef struct {
  long G;
  double tau, s1, s2, d;
} nu_ctx;
static double f_nu(void* c, double v) {
  nu_ctx* k = (nu_ctx*)c;
  return orc_log_fc_nu(v, k->G, k->tau, k->s1, k->s2, k->d);
}
typedef struct {
  long G;
  double ss, sb;
} sig_ctx;
static double f_sig(void* c, double v) {
  sig_ctx* k = (sig_ctx*)c;
  return orc_log_fc_sigma(v, k->G, k->ss, k->sb);
}
/* grouped beta density, P:src/engine.cpp:303-316 */
typedef struct {
  double a, theta, sig2;
  double xi; /* > 0: xi column, prior variance sig2 * xi (extension) */
  long J;
  const orc_group* groups;
  const double* S;
  const double* logS;
  uint64_t* clamps;
} beta_ctx;
static double f_beta(void* c, double b) {
  beta_ctx* k = (beta_ctx*)c;
  double tot = k->a * b;
  for (long j = 0; j < k->J; ++j) {
    const double t = k->groups[j].value * b;
    if (k->logS[j] + t > kExpClamp) {
      if (k->clamps) ++*k->clamps;
      tot -= exp(kExpClamp);
    } else if (k->S[j] > 0.0) {
      tot -= k->S[j] * exp(t);
    }
  }
  const double zz = b - k->theta;
  if (k->xi > 0.0) return tot - zz * zz / (2.0 * (k->sig2 * k->xi));
  return tot - zz * zz / (2.0 * k->sig2);
}
typedef struct {
  int prior;
  double q, k;
} xi_ctx;
static double f_xi(void* c, double x) {
  xi_ctx* k = (xi_ctx*)c;
  return orc_log_fc_xi(k->prior, x, k->q, k->k);
}

/* GibbsEngine::iterate, P:src/engine.cpp:161-370, executed sequentially
 * (the reference result is bitwise independent of worker count). */
int orc_iterate(const orc_engine* e, double* st, double* tw, double* ta,
                long chain, long m, uint64_t* clamps, cmc_error* err) {
  const long G = e->G, N = e->N, L = e->L;
  const uint64_t seed = e->cfg.seed, ch = (uint64_t)chain, it = (uint64_t)m;
  const orc_slice_cfg* sc = &e->scfg;
  const int direct = e->cfg.sampler_mode == CMC_CONJUGATE_DIRECT;
  double* eps = st + ST_EPS(e);
  double* gam = st + ST_GAMMA(e);
  double* beta = st + ST_BETA(e);
  double* theta = st + ST_THETA(e);
  double* sigma = st + ST_SIGMA(e);
  double* nu = st + ST_NU(e);
  double* tau = st + ST_TAU(e);
  double* xi = e->xi_any ? st + ST_XI(e) : NULL;
  double* xb = (double*)malloc(sizeof(double) * (size_t)(G * N));
  double* lp = (double*)malloc(sizeof(double) * (size_t)(G * N));
  double* tmp = (double*)calloc((size_t)G, sizeof(double));
  int rc = CMC_OK;
  int stalled = 0;

  /* refresh_xb, P:src/engine.cpp:144-159 */
  for (long g = 0; g < G; ++g)
    for (long n = 0; n < N; ++n) {
      double acc = 0.0;
      for (long l = 0; l < L; ++l) acc += e->X[n * L + l] * beta[g * L + l];
      xb[g * N + n] = acc;
    }

  /* Step 1: eps, P:src/engine.cpp:178-202 */
  for (long g = 0; g < G; ++g) {
    for (long n = 0; n < N; ++n) {
      orc_stream rng;
      orc_stream_init(&rng, seed, ch, it, site_id(kEps, (uint64_t)(g * N + n)));
      eps_ctx k = {e->y[g * N + n], e->h[n], xb[g * N + n], gam[g], clamps};
      const double x0 = eps[g * N + n];
      const double wv = tw[TU_EPS(e) + g * N + n];
      eps[g * N + n] = orc_slice_step(f_eps, &k, x0, &tw[TU_EPS(e) + g * N + n],
                                      &ta[TU_EPS(e) + g * N + n], sc, m, &rng, &stalled);
      if (stalled) {
        set_stall(err, "epsilon", g + 1, n + 1, x0, wv, m);
        rc = CMC_ERR_STALL;
        goto done;
      }
    }
  }

  /* Step 2: gamma, P:src/engine.cpp:204-226 */
  for (long g = 0; g < G; ++g) {
    ig_ctx k;
    orc_gamma_fc_params(*nu, *tau, eps + g * N, N, &k.shape, &k.scale);
    orc_stream rng;
    orc_stream_init(&rng, seed, ch, it, site_id(kGamma, (uint64_t)g));
    if (direct) {
      gam[g] = 1.0 / orc_gamma(&rng, k.shape, k.scale);
    } else {
      const double x0 = gam[g], wv = tw[TU_GAMMA(e) + g];
      gam[g] = orc_slice_step(f_ig, &k, x0, &tw[TU_GAMMA(e) + g],
                              &ta[TU_GAMMA(e) + g], sc, m, &rng, &stalled);
      if (stalled) {
        set_stall(err, "gamma", g + 1, -1, x0, wv, m);
        rc = CMC_ERR_STALL;
        goto done;
      }
    }
  }

  /* Step 3: nu, P:src/engine.cpp:228-248 */
  for (long g = 0; g < G; ++g) tmp[g] = log(gam[g]);
  const double s1 = orc_det_sum(tmp, G);
  for (long g = 0; g < G; ++g) tmp[g] = 1.0 / gam[g];
  const double s2 = orc_det_sum(tmp, G);
  {
    orc_stream rng;
    orc_stream_init(&rng, seed, ch, it, site_id(kNu, 0));
    nu_ctx k = {G, *tau, s1, s2, e->d};
    const double x0 = *nu, wv = tw[TU_NU(e)];
    *nu = orc_slice_step(f_nu, &k, x0, &tw[TU_NU(e)], &ta[TU_NU(e)], sc, m,
                         &rng, &stalled);
    if (stalled) {
      set_stall(err, "nu", -1, -1, x0, wv, m);
      rc = CMC_ERR_STALL;
      goto done;
    }
  }

  /* Step 4: tau, P:src/engine.cpp:250-267 */
  {
    ig_ctx k;
    orc_tau_fc_params(e->a, e->b, G, *nu, s2, &k.shape, &k.scale);
    orc_stream rng;
    orc_stream_init(&rng, seed, ch, it, site_id(kTau, 0));
    if (direct) {
      *tau = orc_gamma(&rng, k.shape, k.scale);
    } else {
      const double x0 = *tau, wv = tw[TU_TAU(e)];
      *tau = orc_slice_step(f_gr, &k, x0, &tw[TU_TAU(e)], &ta[TU_TAU(e)], sc,
                            m, &rng, &stalled);
      if (stalled) {
        set_stall(err, "tau", -1, -1, x0, wv, m);
        rc = CMC_ERR_STALL;
        goto done;
      }
    }
  }

  /* Step 5: beta columns, P:src/engine.cpp:269-334 */
  for (long g = 0; g < G; ++g)
    for (long n = 0; n < N; ++n)
      lp[g * N + n] = e->h[n] + eps[g * N + n] + xb[g * N + n];
  for (long l = 0; l < L; ++l) {
    const long J = e->n_groups[l];
    const orc_group* grp = e->groups[l];
    const double theta_l = theta[l];
    const double sig2 = sigma[l] * sigma[l];
    double S[64], logS[64];
    double* Sp = J <= 64 ? S : (double*)malloc(sizeof(double) * (size_t)J);
    double* logSp = J <= 64 ? logS : (double*)malloc(sizeof(double) * (size_t)J);
    for (long g = 0; g < G && !stalled; ++g) {
      double* lpg = lp + g * N;
      const double bold = beta[g * L + l];
      for (long j = 0; j < J; ++j) {
        double sacc = 0.0;
        for (long q = 0; q < grp[j].n_idx; ++q)
          sacc += orc_clamped_exp(lpg[grp[j].idx[q]] - grp[j].value * bold, clamps);
        Sp[j] = sacc;
        logSp[j] = log(sacc);
      }
      const int xcol = e->prior[l] != CMC_PRIOR_NORMAL;
      beta_ctx k = {e->A[g * L + l], theta_l, sig2, xcol ? xi[g * L + l] : 0.0,
                    J, grp, Sp, logSp, clamps};
      orc_stream rng;
      orc_stream_init(&rng, seed, ch, it, site_id(kBeta, (uint64_t)(g * L + l)));
      const double wv = tw[TU_BETA(e) + g * L + l];
      const double bnew =
          orc_slice_step(f_beta, &k, bold, &tw[TU_BETA(e) + g * L + l],
                         &ta[TU_BETA(e) + g * L + l], sc, m, &rng, &stalled);
      if (stalled) {
        set_stall(err, "beta", g + 1, l + 1, bold, wv, m);
        rc = CMC_ERR_STALL;
        break;
      }
      beta[g * L + l] = bnew;
      if (bnew != bold)
        for (long j = 0; j < J; ++j)
          for (long q = 0; q < grp[j].n_idx; ++q)
            lpg[grp[j].idx[q]] += grp[j].value * (bnew - bold);
      if (xcol) {
        /* xi_gl right after beta_gl (extension; its conditional reads only
         * beta_gl, theta_l and sigma_l of iteration m-1) */
        const double dz = bnew - theta_l;
        xi_ctx kx = {e->prior[l], dz * dz / (2.0 * sig2), e->t_df};
        orc_stream rx;
        orc_stream_init(&rx, seed, ch, it, site_id(kXi, (uint64_t)(g * L + l)));
        const double x0 = xi[g * L + l], wx = tw[TU_XI(e) + g * L + l];
        xi[g * L + l] = orc_slice_step(f_xi, &kx, x0, &tw[TU_XI(e) + g * L + l],
                                       &ta[TU_XI(e) + g * L + l], sc, m, &rx, &stalled);
        if (stalled) {
          set_stall(err, "xi", g + 1, l + 1, x0, wx, m);
          rc = CMC_ERR_STALL;
          break;
        }
      }
    }
    if (J > 64) {
      free(Sp);
      free(logSp);
    }
    if (stalled) goto done;
  }

  /* Step 6: theta, P:src/engine.cpp:336-347 */
  for (long l = 0; l < L; ++l) {
    double mean, sd;
    if (e->prior[l] != CMC_PRIOR_NORMAL) {
      /* extension: precision 1/c^2 + sum_g 1/(sigma^2 xi_g), mean from
       * sum_g beta_g / xi_g */
      for (long g = 0; g < G; ++g) tmp[g] = 1.0 / xi[g * L + l];
      const double sw = orc_det_sum(tmp, G);
      for (long g = 0; g < G; ++g) tmp[g] = beta[g * L + l] / xi[g * L + l];
      const double sbw = orc_det_sum(tmp, G);
      const double sg = sigma[l], cl = e->c[l];
      const double v = 1.0 / (1.0 / (cl * cl) + sw / (sg * sg));
      mean = v * sbw / (sg * sg);
      sd = sqrt(v);
    } else {
      for (long g = 0; g < G; ++g) tmp[g] = beta[g * L + l];
      const double sb = orc_det_sum(tmp, G);
      orc_theta_fc_params(sb, G, sigma[l], e->c[l], &mean, &sd);
    }
    orc_stream rng;
    orc_stream_init(&rng, seed, ch, it, site_id(kTheta, (uint64_t)l));
    theta[l] = mean + sd * orc_normal(&rng);
  }

  /* Step 7: sigma, P:src/engine.cpp:349-369 */
  for (long l = 0; l < L; ++l) {
    const double th = theta[l];
    const int xcol = e->prior[l] != CMC_PRIOR_NORMAL;
    for (long g = 0; g < G; ++g) {
      const double dlt = beta[g * L + l] - th;
      tmp[g] = xcol ? dlt * dlt / xi[g * L + l] : dlt * dlt;
    }
    sig_ctx k = {G, orc_det_sum(tmp, G), e->s[l]};
    orc_stream rng;
    orc_stream_init(&rng, seed, ch, it, site_id(kSigma, (uint64_t)l));
    const double x0 = sigma[l], wv = tw[TU_SIGMA(e) + l];
    sigma[l] = orc_slice_step(f_sig, &k, x0, &tw[TU_SIGMA(e) + l],
                              &ta[TU_SIGMA(e) + l], sc, m, &rng, &stalled);
    if (stalled) {
      set_stall(err, "sigma", l + 1, -1, x0, wv, m);
      rc = CMC_ERR_STALL;
      goto done;
    }
  }

done:
  free(xb);
  free(lp);
  free(tmp);
  return rc;
}

/* param_value, P:src/streaming.cpp:22-39 */
static double param_value(const orc_engine* e, const double* st, int fam,
                          int idx, long g) {
  switch (fam) {
    case CMC_FAM_BETA_COL: return st[ST_BETA(e) + g * e->L + idx];
    case CMC_FAM_GAMMA: return st[ST_GAMMA(e) + g];
    case CMC_FAM_THETA: return st[ST_THETA(e) + idx];
    case CMC_FAM_SIGMA: return st[ST_SIGMA(e) + idx];
    case CMC_FAM_NU: return st[ST_NU(e)];
    case CMC_FAM_TAU: return st[ST_TAU(e)];
  }
  return 0.0;
}

/* GibbsEngine::run_chain, P:src/engine.cpp:378-455 */
int orc_run_chain(const orc_engine* e, long chain, const cmc_output_view* out,
                  cmc_error* err) {
  const long G = e->G, N = e->N, L = e->L;
  const long XI = e->xi_any ? G * L : 0;
  const long S = G * N + G + G * L + 2 * L + 2 + XI;
  const long T = G * N + G + G * L + L + 2 + XI;
  const long A = 2 + 2 * L + G * L + G + G * N + XI;
  const long ncols = 2 + 2 * L + e->n_saved * (L + 1);
  const long nrows = e->cfg.iterations / e->cfg.thin;
  double* st = (double*)malloc(sizeof(double) * (size_t)S);
  double* tw = (double*)malloc(sizeof(double) * (size_t)T);
  double* ta = (double*)calloc((size_t)T, sizeof(double));
  orc_moments* acc = (orc_moments*)calloc((size_t)A, sizeof(orc_moments));
  long n_prob = 0;
  for (int ci = 0; ci < e->n_contrasts; ++ci)
    n_prob += e->contrasts[ci].per_gene ? G : 1;
  double* prob = (double*)calloc((size_t)(n_prob > 0 ? n_prob : 1), sizeof(double));
  long ccount = 0;
  long row = 0;
  uint64_t clamps = 0;
  int rc = CMC_OK;
  orc_initial_state(e, chain, st);
  for (long i = 0; i < T; ++i) tw[i] = e->cfg.w_init;

  const long total = e->cfg.burnin + e->cfg.iterations;
  for (long m = 1; m <= total; ++m) {
    rc = orc_iterate(e, st, tw, ta, chain, m, &clamps, err);
    if (rc != CMC_OK) break;
    if (m > e->cfg.burnin) {
      /* accumulator order [nu|tau|theta|sigma|beta|gamma|eps] */
      long k = 0;
      orc_moments_update(&acc[k++], st[ST_NU(e)]);
      orc_moments_update(&acc[k++], st[ST_TAU(e)]);
      for (long l = 0; l < L; ++l) orc_moments_update(&acc[k++], st[ST_THETA(e) + l]);
      for (long l = 0; l < L; ++l) orc_moments_update(&acc[k++], st[ST_SIGMA(e) + l]);
      for (long i = 0; i < G * L; ++i) orc_moments_update(&acc[k++], st[ST_BETA(e) + i]);
      for (long g = 0; g < G; ++g) orc_moments_update(&acc[k++], st[ST_GAMMA(e) + g]);
      for (long i = 0; i < G * N; ++i) orc_moments_update(&acc[k++], st[ST_EPS(e) + i]);
      for (long i = 0; i < XI; ++i) orc_moments_update(&acc[k++], st[ST_XI(e) + i]);
      /* ContrastAccumulator::update, P:src/streaming.cpp:90-108 */
      ++ccount;
      const double mc = (double)ccount;
      long off = 0;
      for (int ci = 0; ci < e->n_contrasts; ++ci) {
        const orc_contrast* oc = &e->contrasts[ci];
        const long ng = oc->per_gene ? G : 1;
        for (long g = 0; g < ng; ++g) {
          int all = 1;
          for (int ti = 0; ti < oc->n_terms; ++ti) {
            double lhs = 0.0;
            for (int q = 0; q < oc->n_coefs[ti]; ++q)
              lhs += oc->coef[ti][q] *
                     param_value(e, st, oc->family[ti][q], oc->index[ti][q], g);
            if (!(lhs > oc->threshold[ti])) {
              all = 0;
              break;
            }
          }
          const double ind = all ? 1.0 : 0.0;
          prob[off + g] += (ind - prob[off + g]) / mc;
        }
        off += ng;
      }
      /* thinning, P:src/engine.cpp:433-447 */
      if ((m - e->cfg.burnin) % e->cfg.thin == 0 && row < nrows) {
        if (out->sample_iters) out->sample_iters[row] = m;
        if (out->samples) {
          long col = 0;
          out->samples[(col++) * nrows + row] = st[ST_NU(e)];
          out->samples[(col++) * nrows + row] = st[ST_TAU(e)];
          for (long l = 0; l < L; ++l) out->samples[(col++) * nrows + row] = st[ST_THETA(e) + l];
          for (long l = 0; l < L; ++l) out->samples[(col++) * nrows + row] = st[ST_SIGMA(e) + l];
          for (long s2 = 0; s2 < e->n_saved; ++s2) {
            const long g = e->saved[s2];
            for (long l = 0; l < L; ++l)
              out->samples[(col++) * nrows + row] = st[ST_BETA(e) + g * L + l];
            out->samples[(col++) * nrows + row] = st[ST_GAMMA(e) + g];
          }
          (void)ncols;
        }
        ++row;
      }
    }
  }
  if (rc == CMC_OK) {
    if (out->acc_count) *out->acc_count = acc[0].count;
    for (long i = 0; i < A; ++i) {
      if (out->acc_mean) out->acc_mean[i] = acc[i].mean;
      if (out->acc_meansq) out->acc_meansq[i] = acc[i].meansq;
      if (out->acc_mean_c) out->acc_mean_c[i] = acc[i].mean_c;
      if (out->acc_meansq_c) out->acc_meansq_c[i] = acc[i].meansq_c;
    }
    if (out->contrast_prob)
      for (long i = 0; i < n_prob; ++i) out->contrast_prob[i] = prob[i];
    if (out->contrast_count)
      for (int ci = 0; ci < e->n_contrasts; ++ci) out->contrast_count[ci] = ccount;
    if (out->clamp_events) *out->clamp_events = clamps;
    if (out->final_state)
      for (long i = 0; i < S; ++i) out->final_state[i] = st[i];
  }
  free(st);
  free(tw);
  free(ta);
  free(acc);
  free(prob);
  return rc;
}
