// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference countmc library, compiled
// from /root/reference/proj/src/*.cpp by oracle/Makefile into
// oracle/_ref/libcountmc_ref.so.  It lets the tests (bit-for-bit parity) and
// bench.py's reference arm / cpu_baseline drive the reference's own public
// API (GibbsEngine, P:include/countmc/engine.hpp:110-159) with the same
// packed arrays the product uses (include/countmc_b200.h).  No reference
// source is copied: this file only includes the reference headers.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "countmc/diagnostics.hpp"
#include "countmc/engine.hpp"
#include "countmc/errors.hpp"
#include "countmc/io.hpp"
#include "countmc/model.hpp"
#include "countmc/parallel.hpp"
#include "countmc/rng.hpp"
#include "countmc/simulate.hpp"
#include "countmc/slice.hpp"
#include "countmc/streaming.hpp"
#include "countmc/types.hpp"

#include "../include/countmc_b200.h"

using namespace countmc;

namespace {

struct RefEngine {
  CountMatrix data;
  ModelSpec spec;
  std::unique_ptr<GibbsEngine> engine;
  long G, N, L;
};

void fill_err(cmc_error* err, int code, const char* msg) {
  if (!err) return;
  std::memset(err, 0, sizeof(*err));
  err->code = code;
  err->index1 = err->index2 = -1;
  std::snprintf(err->msg, sizeof(err->msg), "%s", msg);
}

void fill_stall(cmc_error* err, const SamplerStallError& e) {
  if (!err) return;
  std::memset(err, 0, sizeof(*err));
  err->code = CMC_ERR_STALL;
  std::snprintf(err->step, sizeof(err->step), "%s", e.step().c_str());
  err->index1 = e.index1();
  err->index2 = e.index2();
  err->x0 = e.x0();
  err->width = e.width();
  err->iteration = e.iteration();
  std::snprintf(err->msg, sizeof(err->msg), "%s", e.what());
}

RunConfig to_cfg(const cmc_run_config* c) {
  RunConfig r;
  r.chains = c->chains;
  r.iterations = c->iterations;
  r.burnin = c->burnin;
  r.tune_cutoff = c->tune_cutoff;
  r.thin = c->thin;
  r.seed = c->seed;
  r.slice.max_step_out = c->max_step_out;
  r.slice.max_shrink = c->max_shrink;
  r.slice.w_init = c->w_init;
  r.save_genes = c->save_genes;
  r.workers = c->workers;
  r.sampler_mode = c->sampler_mode == CMC_CONJUGATE_DIRECT
                       ? SamplerMode::conjugate_direct
                       : SamplerMode::slice_faithful;
  r.concurrent_chains = c->concurrent_chains != 0;
  return r;
}

std::vector<ContrastSpec> to_contrasts(const cmc_contrast_set* cs) {
  std::vector<ContrastSpec> out;
  if (!cs) return out;
  int t = 0, q = 0;
  for (int ci = 0; ci < cs->n_contrasts; ++ci) {
    ContrastSpec spec;
    spec.id = "c" + std::to_string(ci + 1);
    for (int ti = 0; ti < cs->n_terms[ci]; ++ti, ++t) {
      ContrastTerm term;
      term.threshold = cs->threshold[t];
      for (int k = 0; k < cs->n_coefs[t]; ++k, ++q) {
        ParamRef ref;
        ref.family = static_cast<ParamFamily>(cs->family[q]);
        ref.index = static_cast<std::size_t>(cs->index[q]);
        term.coeffs.push_back({ref, cs->coef[q]});
      }
      spec.terms.push_back(term);
    }
    out.push_back(spec);
  }
  return out;
}

void unpack_state(const RefEngine* r, const double* p, ChainState& st) {
  const long G = r->G, N = r->N, L = r->L;
  st = ChainState(G, N, L);
  std::memcpy(st.eps.data().data(), p, sizeof(double) * G * N);
  p += G * N;
  std::memcpy(st.gamma.data(), p, sizeof(double) * G);
  p += G;
  std::memcpy(st.beta.data().data(), p, sizeof(double) * G * L);
  p += G * L;
  std::memcpy(st.theta.data(), p, sizeof(double) * L);
  p += L;
  std::memcpy(st.sigma.data(), p, sizeof(double) * L);
  p += L;
  st.nu = p[0];
  st.tau = p[1];
}

void pack_state(const RefEngine* r, const ChainState& st, double* p) {
  const long G = r->G, N = r->N, L = r->L;
  std::memcpy(p, st.eps.data().data(), sizeof(double) * G * N);
  p += G * N;
  std::memcpy(p, st.gamma.data(), sizeof(double) * G);
  p += G;
  std::memcpy(p, st.beta.data().data(), sizeof(double) * G * L);
  p += G * L;
  std::memcpy(p, st.theta.data(), sizeof(double) * L);
  p += L;
  std::memcpy(p, st.sigma.data(), sizeof(double) * L);
  p += L;
  p[0] = st.nu;
  p[1] = st.tau;
}

void unpack_tuning(const RefEngine* r, const double* w, const double* a,
                   TuningState& t) {
  const long G = r->G, N = r->N, L = r->L;
  t = TuningState(G, N, L, 1.0);
  long k = 0;
  auto take = [&](SliceVar& v) {
    v.w = w[k];
    v.w_aux = a[k];
    ++k;
  };
  for (auto& v : t.eps) take(v);
  for (auto& v : t.gamma) take(v);
  for (auto& v : t.beta) take(v);
  for (auto& v : t.sigma) take(v);
  take(t.nu);
  take(t.tau);
}

void pack_tuning(const RefEngine* r, const TuningState& t, double* w,
                 double* a) {
  (void)r;
  long k = 0;
  auto put = [&](const SliceVar& v) {
    w[k] = v.w;
    a[k] = v.w_aux;
    ++k;
  };
  for (auto& v : t.eps) put(v);
  for (auto& v : t.gamma) put(v);
  for (auto& v : t.beta) put(v);
  for (auto& v : t.sigma) put(v);
  put(t.nu);
  put(t.tau);
}

void copy_moments(const MomentAccumulator& m, long i, const cmc_output_view* o) {
  if (o->acc_mean) o->acc_mean[i] = m.mean();
  if (o->acc_meansq) o->acc_meansq[i] = m.meansq();
}

void write_output(const RefEngine* r, const ChainOutput& co,
                  const cmc_output_view* o) {
  const long G = r->G, N = r->N, L = r->L;
  long k = 0;
  if (o->acc_count) *o->acc_count = co.nu_acc.count();
  copy_moments(co.nu_acc, k++, o);
  copy_moments(co.tau_acc, k++, o);
  for (long l = 0; l < L; ++l) copy_moments(co.theta_acc[l], k++, o);
  for (long l = 0; l < L; ++l) copy_moments(co.sigma_acc[l], k++, o);
  for (long i = 0; i < G * L; ++i) copy_moments(co.beta_acc[i], k++, o);
  for (long g = 0; g < G; ++g) copy_moments(co.gamma_acc[g], k++, o);
  for (long i = 0; i < G * N; ++i) copy_moments(co.eps_acc[i], k++, o);
  long off = 0;
  for (std::size_t ci = 0; ci < co.contrasts.size(); ++ci) {
    const auto& p = co.contrasts[ci].prob();
    if (o->contrast_prob)
      for (std::size_t g = 0; g < p.size(); ++g) o->contrast_prob[off + g] = p[g];
    off += static_cast<long>(p.size());
    if (o->contrast_count) o->contrast_count[ci] = co.contrasts[ci].count();
  }
  const long nrows = static_cast<long>(co.sample_iters.size());
  if (o->samples)
    for (std::size_t c = 0; c < co.samples.size(); ++c)
      for (long rr = 0; rr < nrows; ++rr)
        o->samples[c * nrows + rr] = co.samples[c][rr];
  if (o->sample_iters)
    for (long rr = 0; rr < nrows; ++rr) o->sample_iters[rr] = co.sample_iters[rr];
  if (o->clamp_events) *o->clamp_events = co.clamp_events;
  if (o->final_state) pack_state(r, co.final_state, o->final_state);
  if (o->step_seconds)
    for (int s = 0; s < 7; ++s) o->step_seconds[s] = co.timings.seconds[s];
}

}  // namespace

extern "C" {

int ref_engine_create(const cmc_problem* p, const cmc_run_config* c,
                      const cmc_contrast_set* cs, void** out, cmc_error* err) {
  *out = nullptr;
  auto* r = new RefEngine();
  r->G = p->G;
  r->N = p->N;
  r->L = p->L;
  try {
    r->data.counts = Grid<long long>(p->G, p->N, 0);
    std::memcpy(r->data.counts.data().data(), p->counts,
                sizeof(long long) * p->G * p->N);
    for (long g = 0; g < p->G; ++g) r->data.genes.push_back("g" + std::to_string(g + 1));
    for (long n = 0; n < p->N; ++n) r->data.samples.push_back("s" + std::to_string(n + 1));
    r->spec.X = Matrix(p->N, p->L, 0.0);
    std::memcpy(r->spec.X.data().data(), p->X, sizeof(double) * p->N * p->L);
    r->spec.h.assign(p->h, p->h + p->N);
    r->spec.priors.a = p->a;
    r->spec.priors.b = p->b;
    r->spec.priors.d = p->d;
    r->spec.priors.c.assign(p->c, p->c + p->L);
    r->spec.priors.s.assign(p->s, p->s + p->L);
    r->engine = std::make_unique<GibbsEngine>(r->data, r->spec, to_cfg(c),
                                              to_contrasts(cs));
  } catch (const ConfigError& e) {
    fill_err(err, CMC_ERR_CONFIG, e.what());
    delete r;
    return CMC_ERR_CONFIG;
  } catch (const std::exception& e) {
    fill_err(err, CMC_ERR_ARG, e.what());
    delete r;
    return CMC_ERR_ARG;
  }
  *out = r;
  return CMC_OK;
}

void ref_engine_destroy(void* h) { delete static_cast<RefEngine*>(h); }

long ref_engine_n_saved(void* h) {
  return static_cast<long>(static_cast<RefEngine*>(h)->engine->saved_genes().size());
}

void ref_engine_saved_genes(void* h, long* out) {
  const auto& s = static_cast<RefEngine*>(h)->engine->saved_genes();
  for (std::size_t i = 0; i < s.size(); ++i) out[i] = static_cast<long>(s[i]);
}

long ref_engine_tune_cutoff(void* h) {
  return static_cast<RefEngine*>(h)->engine->config().tune_cutoff;
}

void ref_initial_state(void* h, long chain, double* st) {
  auto* r = static_cast<RefEngine*>(h);
  pack_state(r, r->engine->initial_state(chain), st);
}

int ref_iterate(void* h, double* st, double* tw, double* ta, long chain,
                long m, int workers, uint64_t* clamps, cmc_error* err) {
  auto* r = static_cast<RefEngine*>(h);
  ChainState state;
  TuningState tuning;
  unpack_state(r, st, state);
  unpack_tuning(r, tw, ta, tuning);
  ThreadPool pool(workers);
  EngineScratch scratch(r->G, r->N);
  ClampCounter cc;
  int rc = CMC_OK;
  try {
    r->engine->iterate(state, tuning, chain, m, pool, scratch, &cc);
  } catch (const SamplerStallError& e) {
    fill_stall(err, e);
    rc = CMC_ERR_STALL;
  }
  if (clamps) *clamps += cc.count();
  pack_state(r, state, st);
  pack_tuning(r, tuning, tw, ta);
  return rc;
}

// GibbsEngine::run() (P:src/engine.cpp:457-483); outputs[c] per chain.
int ref_run(void* h, const cmc_output_view* outputs, cmc_error* err) {
  auto* r = static_cast<RefEngine*>(h);
  try {
    const auto outs = r->engine->run();
    for (std::size_t c = 0; c < outs.size(); ++c) write_output(r, outs[c], &outputs[c]);
  } catch (const SamplerStallError& e) {
    fill_stall(err, e);
    return CMC_ERR_STALL;
  }
  return CMC_OK;
}

// The reference's own run() + write_results (P:src/io.cpp:571-720) into
// outdir; genes (G labels) may be NULL (keeps "g<g+1>").  Returns the
// seconds write_results took in *write_s.
int ref_write_results(void* h, const char* outdir, const char* const* genes,
                      double wall_seconds, double* write_s, cmc_error* err) {
  auto* r = static_cast<RefEngine*>(h);
  try {
    if (genes)
      for (long g = 0; g < r->G; ++g) r->data.genes[g] = genes[g];
    const auto outs = r->engine->run();
    const auto t0 = std::chrono::steady_clock::now();
    write_results(outdir, r->data, r->spec, r->engine->config(), outs, wall_seconds);
    *write_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  } catch (const SamplerStallError& e) {
    fill_stall(err, e);
    return CMC_ERR_STALL;
  } catch (const ConfigError& e) {
    fill_err(err, CMC_ERR_CONFIG, e.what());
    return CMC_ERR_CONFIG;
  }
  return CMC_OK;
}

// CPU baseline: the reference's own iterate() plus run_chain's monitored
// loop body (P:src/engine.cpp:409-431: moment and contrast accumulators),
// `burn` un-timed burn-in sweeps then `sweeps` timed sweeps on `workers`
// threads.  Returns wall seconds of the timed sweeps.
double ref_bench_chains(void* h, int burn_workers, int workers, long chains, long burn,
                        long sweeps);

double ref_bench(void* h, int workers, long burn, long sweeps) {
  return ref_bench_chains(h, workers, workers, 1, burn, sweeps);
}

// Burn-in on burn_workers threads, then `sweeps` monitored sweeps timed on
// `workers` threads (iterate is bitwise independent of the worker count).
// `chains` chains run one after another, as run() runs them (chains in
// sequence on one pool, P:src/engine.cpp:457-483); the timed seconds of
// every chain's monitored sweeps are summed.
double ref_bench_chains(void* h, int burn_workers, int workers, long chains, long burn,
                        long sweeps) {
  auto* r = static_cast<RefEngine*>(h);
  const auto& cfg = r->engine->config();
  const long G = r->G, N = r->N, L = r->L;
  double total = 0.0;
  for (long c = 0; c < chains; ++c) {
    ChainState state = r->engine->initial_state(c);
    TuningState tuning(G, N, L, cfg.slice.w_init);
    EngineScratch scratch(G, N);
    ClampCounter clamps;
    std::vector<MomentAccumulator> theta_acc(L), sigma_acc(L), beta_acc(G * L),
        gamma_acc(G), eps_acc(G * N);
    MomentAccumulator nu_acc, tau_acc;
    std::vector<ContrastAccumulator> contrasts;
    for (const auto& spec : r->engine->contrast_specs()) contrasts.emplace_back(spec, G);
    {
      ThreadPool burn_pool(burn_workers);
      for (long m = 1; m <= burn; ++m)
        r->engine->iterate(state, tuning, c, m, burn_pool, scratch, &clamps);
    }
    ThreadPool pool(workers);
    const auto t0 = std::chrono::steady_clock::now();
    for (long m = burn + 1; m <= burn + sweeps; ++m) {
      r->engine->iterate(state, tuning, c, m, pool, scratch, &clamps);
      nu_acc.update(state.nu);
      tau_acc.update(state.tau);
      for (long l = 0; l < L; ++l) {
        theta_acc[l].update(state.theta[l]);
        sigma_acc[l].update(state.sigma[l]);
      }
      pool.parallel_for(G, std::max<long>(1, G / (8 * pool.workers())),
                        [&](long g0, long g1) {
                          for (long g = g0; g < g1; ++g) {
                            for (long l = 0; l < L; ++l)
                              beta_acc[g * L + l].update(state.beta(g, l));
                            gamma_acc[g].update(state.gamma[g]);
                            const double* eps = state.eps.row(g);
                            for (long n = 0; n < N; ++n) eps_acc[g * N + n].update(eps[n]);
                          }
                        });
      for (auto& acc : contrasts) acc.update(state);
    }
    const auto t1 = std::chrono::steady_clock::now();
    total += std::chrono::duration<double>(t1 - t0).count();
  }
  return total;
}

double ref_bench_split(void* h, int burn_workers, int workers, long burn, long sweeps) {
  return ref_bench_chains(h, burn_workers, workers, 1, burn, sweeps);
}

// build_diagnostics (P:src/io.cpp:507-569) numerics with the reference's
// own gelman_rhat / credible_interval / effective_sample_size
// (P:src/diagnostics.cpp), after GibbsEngine::run().  Row order
// [nu|tau|theta|sigma|beta g-major|gamma]; ESS per retained column.
int ref_diagnostics(void* h, double* rhat, int* flags, double* mean, double* sd,
                    double* lo, double* hi, double* ess, int* ess_status, cmc_error* err) {
  auto* r = static_cast<RefEngine*>(h);
  std::vector<ChainOutput> outs;
  try {
    outs = r->engine->run();
  } catch (const SamplerStallError& e) {
    fill_stall(err, e);
    return CMC_ERR_STALL;
  }
  const long G = r->G, L = r->L;
  long row = 0;
  auto one = [&](auto&& get) {
    std::vector<MomentAccumulator> accs;
    for (const auto& ch : outs) accs.push_back(get(ch));
    const RhatResult rr = gelman_rhat(accs);
    rhat[row] = rr.value;
    double pm = 0.0, pms = 0.0;
    for (const auto& a : accs) {
      pm += a.mean();
      pms += a.meansq();
    }
    pm /= static_cast<double>(accs.size());
    pms /= static_cast<double>(accs.size());
    const double var = std::max(0.0, pms - pm * pm);
    const Interval ci = credible_interval(pm, pms, 0.05);
    mean[row] = pm;
    sd[row] = std::sqrt(var);
    lo[row] = ci.lo;
    hi[row] = ci.hi;
    flags[row] = (rr.degenerate ? 1 : 0) | ((rr.degenerate || rr.value < 1.1) ? 2 : 0);
    ++row;
  };
  one([](const ChainOutput& c) { return c.nu_acc; });
  one([](const ChainOutput& c) { return c.tau_acc; });
  for (long l = 0; l < L; ++l) one([l](const ChainOutput& c) { return c.theta_acc[l]; });
  for (long l = 0; l < L; ++l) one([l](const ChainOutput& c) { return c.sigma_acc[l]; });
  for (long g = 0; g < G; ++g)
    for (long l = 0; l < L; ++l)
      one([g, l, L](const ChainOutput& c) { return c.beta_acc[g * L + l]; });
  for (long g = 0; g < G; ++g) one([g](const ChainOutput& c) { return c.gamma_acc[g]; });
  const std::size_t ncol = outs[0].samples.size();
  for (std::size_t col = 0; col < ncol; ++col) {
    std::vector<std::vector<double>> series;
    for (const auto& ch : outs) series.push_back(ch.samples[col]);
    const EssResult e = effective_sample_size(series);
    ess[col] = e.value;
    ess_status[col] = e.status == EssResult::Status::ok ? 0
                      : e.status == EssResult::Status::undefined ? 1 : 2;
  }
  return CMC_OK;
}

// ---- input side: load_counts (P:src/io.cpp:125-164), estimate_offsets
// (P:src/model.cpp:21-68).  Returns 0, 6 (LoadError), 1 (ConfigError) or
// -1 when cells/names capacity is short (G, N still written).  Names are
// NUL-separated: samples first, then genes.
int ref_load_counts(const char* path, long long* cells, long cap_cells, char* names,
                    long cap_names, long* G, long* N, int* dup, char* msg) {
  try {
    const CountMatrix m = load_counts(path);
    *G = static_cast<long>(m.G());
    *N = static_cast<long>(m.N());
    *dup = m.duplicate_genes ? 1 : 0;
    std::string all;
    for (const auto& s : m.samples) all.append(s).push_back('\0');
    for (const auto& g : m.genes) all.append(g).push_back('\0');
    if (cap_cells < *G * *N || cap_names < static_cast<long>(all.size())) return -1;
    std::memcpy(cells, m.counts.data().data(), sizeof(long long) * m.counts.data().size());
    std::memcpy(names, all.data(), all.size());
    return 0;
  } catch (const LoadError& e) {
    std::snprintf(msg, 256, "%s", e.what());
    return 6;
  } catch (const ConfigError& e) {
    std::snprintf(msg, 256, "%s", e.what());
    return 1;
  }
}

// load_model_matrix / load_offsets (P:src/io.cpp:178-243): values into
// out (capacity cap), dims in rows/cols; 0, 6 (LoadError) or -1 (capacity).
int ref_load_table(const char* path, int which, double* out, long cap, long* rows, long* cols,
                   char* msg) {
  try {
    std::vector<double> v;
    if (which == 0) {
      const DesignTable t = load_model_matrix(path);
      *rows = static_cast<long>(t.X.rows());
      *cols = static_cast<long>(t.X.cols());
      v = t.X.data();
    } else {
      v = load_offsets(path);
      *rows = static_cast<long>(v.size());
      *cols = 1;
    }
    if (cap < static_cast<long>(v.size())) return -1;
    std::memcpy(out, v.data(), sizeof(double) * v.size());
    return 0;
  } catch (const LoadError& e) {
    std::snprintf(msg, 256, "%s", e.what());
    return 6;
  }
}

int ref_estimate_offsets(long G, long N, const long long* counts, double* h, char* msg) {
  CountMatrix m;
  m.counts = Grid<long long>(G, N, 0);
  std::memcpy(m.counts.data().data(), counts, sizeof(long long) * G * N);
  for (long g = 0; g < G; ++g) m.genes.push_back("g" + std::to_string(g));
  for (long n = 0; n < N; ++n) m.samples.push_back("s" + std::to_string(n));
  try {
    const std::vector<double> out = estimate_offsets(m);
    std::memcpy(h, out.data(), sizeof(double) * N);
    return 0;
  } catch (const ConfigError& e) {
    std::snprintf(msg, 256, "%s", e.what());
    return 1;
  }
}

int ref_hardware_threads() {
  return static_cast<int>(std::thread::hardware_concurrency());
}

// ---- primitives for pinning the oracle against the reference itself ----
void ref_philox(const uint64_t* ctr, const uint64_t* key, uint64_t* out) {
  const auto r = philox4x64({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
  for (int i = 0; i < 4; ++i) out[i] = r[i];
}
double ref_normal_quantile(double p) { return normal_quantile(p); }
void ref_stream_u01(uint64_t seed, uint64_t chain, uint64_t it, uint64_t site,
                    long n, double* out) {
  RngStream s(seed, chain, it, site);
  for (long i = 0; i < n; ++i) out[i] = s.u01();
}
void ref_stream_gamma(uint64_t seed, uint64_t site, double shape, double rate,
                      long n, double* out) {
  RngStream s(seed, 0, 0, site);
  for (long i = 0; i < n; ++i) out[i] = s.gamma(shape, rate);
}
double ref_log_fc_epsilon(long long y, double h, double eta, double g, double e) {
  return log_fc_epsilon(y, h, eta, g, e);
}
double ref_log_fc_nu(double nu, long G, double tau, double s1, double s2, double d) {
  return log_fc_nu(nu, G, tau, s1, s2, d);
}
double ref_log_fc_sigma(double s, long G, double ss, double sb) {
  return log_fc_sigma(s, G, ss, sb);
}
double ref_pairwise_sum(const double* x, long n) { return pairwise_sum(x, n); }


// ---- the reference's own synthetic inputs (bench.py's reference arm) ----
// generate() (P:src/simulate.cpp:28-90) with builtin_design (:123-142) when
// X is null; counts out as G x N row-major.  0 ok, 1 ConfigError or
// SimulationError (message in msg).
int ref_generate(long G, long N, long L, const double* X, const double* h, double nu,
                 double tau, const double* theta, const double* sigma, uint64_t seed,
                 long long* counts, char* msg) {
  try {
    SimSpec spec;
    spec.G = (std::size_t)G;
    spec.N = (std::size_t)N;
    if (X) {
      spec.X = Matrix((std::size_t)N, (std::size_t)L, 0.0);
      std::memcpy(spec.X.data().data(), X, sizeof(double) * N * L);
    } else {
      spec.X = builtin_design("heterosis16x5", (std::size_t)N);
    }
    if (h) spec.h.assign(h, h + N);
    spec.nu = nu;
    spec.tau = tau;
    spec.theta.assign(theta, theta + spec.L());
    spec.sigma.assign(sigma, sigma + spec.L());
    spec.seed = seed;
    auto out = generate(spec);
    std::memcpy(counts, out.first.counts.data().data(), sizeof(long long) * G * N);
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(msg, 256, "%s", e.what());
    return 1;
  }
}
void ref_builtin_design(long N, double* X) {
  const Matrix m = builtin_design("heterosis16x5", (std::size_t)N);
  std::memcpy(X, m.data().data(), sizeof(double) * m.size());
}

}  // extern "C"
