/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  A plain-C restatement of the
 * reference countmc Gibbs sweep (/root/reference/proj, cited as P:) used as
 * the parity checker for the CUDA path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it; the
 * product library never links or calls it.
 *
 * Parity pinning: tests/test_oracle_*.py check this restatement against the
 * reference's own known-answer values (P:tests/test_rng.cpp:19-71,152-167,
 * P:tests/test_model.cpp, P:tests/test_slice.cpp, P:tests/test_streaming.cpp,
 * P:tests/test_parallel.cpp) and bit-for-bit against the reference itself,
 * compiled from its sources into oracle/_ref/ (see oracle/Makefile), through
 * committed golden sweeps in tests/golden/.
 *
 * Types come from include/countmc_b200.h so the oracle, the compiled
 * reference shim and the product share one array layout.
 */
#ifndef COUNTMC_ORACLE_H
#define COUNTMC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/countmc_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG (P:src/rng.cpp, P:include/countmc/rng.hpp) ---- */
void orc_philox4x64(const uint64_t ctr[4], const uint64_t key[2],
                    uint64_t out[4]);

typedef struct orc_stream {
  uint64_t ctr[4];
  uint64_t key[2];
  uint64_t buf[4];
  int pos;
} orc_stream;

void orc_stream_init(orc_stream* s, uint64_t seed, uint64_t chain,
                     uint64_t iteration, uint64_t site);
uint64_t orc_next(orc_stream* s);
double orc_u01(orc_stream* s);
uint64_t orc_uniform_int(orc_stream* s, uint64_t n);
double orc_normal(orc_stream* s);
double orc_gamma(orc_stream* s, double shape, double rate);
double orc_normal_quantile(double p);
/* Fills out[i] = u01 of the first n draws of stream (seed, chain, it, site). */
void orc_stream_u01(uint64_t seed, uint64_t chain, uint64_t it, uint64_t site,
                    long n, double* out);

/* ---- model (P:src/model.cpp) ---- */
double orc_clamped_exp(double x, uint64_t* clamps);
double orc_log_fc_epsilon(long long y, double h, double eta, double gamma,
                          double eps, uint64_t* clamps);
void orc_gamma_fc_params(double nu, double tau, const double* eps_row,
                         long N, double* shape, double* scale);
double orc_log_invgamma(double x, double shape, double scale);
double orc_log_gamma_rate(double x, double shape, double rate);
double orc_log_fc_nu(double nu, long G, double tau, double sum_log_gamma,
                     double sum_inv_gamma, double d);
void orc_tau_fc_params(double a, double b, long G, double nu,
                       double sum_inv_gamma, double* shape, double* rate);
void orc_theta_fc_params(double sum_beta, long G, double sigma, double c,
                         double* mean, double* sd);
double orc_log_fc_sigma(double sigma, long G, double ss, double s_bound);
/* extension (no reference): xi full conditional, CMC_PRIOR_* families */
double orc_log_fc_xi(int prior, double xi, double q, double k);

/* ---- slice (P:include/countmc/slice.hpp) ---- */
typedef double (*orc_logf)(void* ctx, double x);
typedef struct orc_slice_cfg {
  int max_step_out;
  long burnin;
  long tune_cutoff;
  double w_init;
  int max_shrink;
} orc_slice_cfg;
void orc_tune_update(double* w, double* w_aux, long m, double delta,
                     const orc_slice_cfg* cfg);
/* Returns the new value; on a stall sets *stalled = 1 and returns x0. */
double orc_slice_step(orc_logf f, void* ctx, double x0, double* w,
                      double* w_aux, const orc_slice_cfg* cfg, long m,
                      orc_stream* rng, int* stalled);
/* Convenience for tests: slice chain on a named density
 * (0: -x^2/2, 1: Gamma(3, rate 2), 2: InvGamma(2, 3), 3: U(0,1) box). */
int orc_slice_chain(int density, double x0, long n, long burnin,
                    double w_init, uint64_t seed, double* out);

/* ---- reductions (P:include/countmc/parallel.hpp:57-84, P:src/parallel.cpp:81-86) ---- */
double orc_pairwise_sum(const double* x, size_t n);
double orc_det_sum(const double* x, long n);

/* ---- streaming (P:include/countmc/streaming.hpp:15-34, P:src/streaming.cpp:90-112) ---- */
typedef struct orc_moments {
  long count;
  double mean, meansq, mean_c, meansq_c;
} orc_moments;
void orc_moments_update(orc_moments* acc, double value);
void orc_moments_stream(const double* v, long n, double* mean, double* meansq);
double orc_disjunction_combine(double p1, double p2, double p12);

/* ---- engine (P:src/engine.cpp) ---- */
typedef struct orc_engine orc_engine;
int orc_engine_create(const cmc_problem* p, const cmc_run_config* cfg,
                      const cmc_contrast_set* contrasts, orc_engine** out,
                      cmc_error* err);
void orc_engine_destroy(orc_engine* e);
int orc_engine_config(const orc_engine* e, cmc_run_config* out);
long orc_engine_n_saved(const orc_engine* e);
int orc_engine_saved_genes(const orc_engine* e, long* out);
int orc_initial_state(const orc_engine* e, long chain, double* state);
int orc_iterate(const orc_engine* e, double* state, double* tun_w,
                double* tun_waux, long chain, long m, uint64_t* clamps,
                cmc_error* err);
int orc_run_chain(const orc_engine* e, long chain, const cmc_output_view* out,
                  cmc_error* err);

#ifdef __cplusplus
}
#endif

#endif
