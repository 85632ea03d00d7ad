// countmc_b200.hpp — header-only C++ facade over the C-ABI, mirroring the
// reference countmc::GibbsEngine interface (P:include/countmc/engine.hpp:
// 110-159) so a C++ caller can switch by changing one include and one
// namespace.  Same member names, argument meaning and exceptions
// (ConfigError / SamplerStallError, P:include/countmc/errors.hpp).
#pragma once

#include <cstdint>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "countmc_b200.h"

namespace countmc_b200 {

class ConfigError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

class SamplerStallError : public std::runtime_error {
 public:
  explicit SamplerStallError(const cmc_error& e)
      : std::runtime_error(e.msg), step_(e.step), index1_(e.index1),
        index2_(e.index2), x0_(e.x0), width_(e.width), iteration_(e.iteration) {}
  const std::string& step() const { return step_; }
  long index1() const { return index1_; }
  long index2() const { return index2_; }
  double x0() const { return x0_; }
  double width() const { return width_; }
  long iteration() const { return iteration_; }

 private:
  std::string step_;
  long index1_, index2_;
  double x0_, width_;
  long iteration_;
};

class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

class LoadError : public std::runtime_error {  // P:include/countmc/errors.hpp:16
 public:
  using std::runtime_error::runtime_error;
};

class NormalizationError : public ConfigError {  // P:include/countmc/errors.hpp:22
 public:
  using ConfigError::ConfigError;
};

inline void check(int rc, const cmc_error& e) {
  if (rc == CMC_OK) return;
  if (rc == CMC_ERR_CONFIG) throw ConfigError(e.msg);
  if (rc == CMC_ERR_STALL) throw SamplerStallError(e);
  if (rc == CMC_ERR_ARG) throw std::invalid_argument(e.msg);
  if (rc == CMC_ERR_LOAD) throw LoadError(e.msg);
  throw DeviceError(e.msg);
}

// CountMatrix (P:include/countmc/types.hpp:50-58): G x N row-major counts.
struct CountMatrix {
  long G = 0, N = 0;
  std::vector<long long> counts;
  std::vector<std::string> genes, samples;
  bool duplicate_genes = false;
};

// load_counts (P:src/io.cpp:125-164), multithreaded; throws LoadError.
inline CountMatrix load_counts(const std::string& path) {
  cmc_counts* h = nullptr;
  cmc_error e{};
  check(cmc_counts_load(path.c_str(), &h, &e), e);
  CountMatrix m;
  int dup = 0;
  cmc_counts_dims(h, &m.G, &m.N, &dup);
  m.duplicate_genes = dup != 0;
  const long long* d = cmc_counts_data(h);
  m.counts.assign(d, d + m.G * m.N);
  for (long g = 0; g < m.G; ++g) m.genes.emplace_back(cmc_counts_gene(h, g));
  for (long n = 0; n < m.N; ++n) m.samples.emplace_back(cmc_counts_sample(h, n));
  cmc_counts_free(h);
  return m;
}

// DesignTable / load_model_matrix (P:src/io.cpp:178-205): X is N x L
// row-major, effects the header labels; throws LoadError.
struct DesignTable {
  long N = 0, L = 0;
  std::vector<double> X;
  std::vector<std::string> effects;
};

inline DesignTable load_model_matrix(const std::string& path) {
  cmc_table* t = nullptr;
  cmc_error e{};
  check(cmc_model_matrix_load(path.c_str(), &t, &e), e);
  DesignTable d;
  cmc_table_dims(t, &d.N, &d.L);
  const double* x = cmc_table_data(t);
  d.X.assign(x, x + d.N * d.L);
  for (long l = 0; l < d.L; ++l) d.effects.emplace_back(cmc_table_name(t, l));
  cmc_table_free(t);
  return d;
}

// load_offsets (P:src/io.cpp:221-243); throws LoadError.
inline std::vector<double> load_offsets(const std::string& path) {
  cmc_table* t = nullptr;
  cmc_error e{};
  check(cmc_offsets_load(path.c_str(), &t, &e), e);
  long n = 0;
  cmc_table_dims(t, &n, nullptr);
  const double* h = cmc_table_data(t);
  std::vector<double> out(h, h + n);
  cmc_table_free(t);
  return out;
}

// estimate_offsets (P:src/model.cpp:21-68), bit-identical; throws
// NormalizationError when no gene is positive in every sample.
inline std::vector<double> estimate_offsets(const CountMatrix& m) {
  std::vector<double> h(static_cast<size_t>(m.N));
  cmc_error e{};
  const int rc = cmc_estimate_offsets(m.G, m.N, m.counts.data(), h.data(), &e);
  if (rc == CMC_ERR_CONFIG) throw NormalizationError(e.msg);
  check(rc, e);
  return h;
}

enum class SamplerMode { slice_faithful, conjugate_direct };

struct SliceConfig {  // P:include/countmc/slice.hpp:11-17
  int max_step_out = 100;
  double w_init = 1.0;
  int max_shrink = 1000;
};

struct RunConfig {  // P:include/countmc/engine.hpp:21-36
  long chains = 4;
  long iterations = 4000;
  long burnin = 2000;
  long tune_cutoff = -1;
  long thin = 20;
  std::uint64_t seed = 1;
  SliceConfig slice;
  long save_genes = 20;
  int workers = 1;
  SamplerMode sampler_mode = SamplerMode::slice_faithful;
  bool concurrent_chains = false;

  cmc_run_config to_c() const {
    cmc_run_config c{};
    c.chains = chains;
    c.iterations = iterations;
    c.burnin = burnin;
    c.tune_cutoff = tune_cutoff;
    c.thin = thin;
    c.seed = seed;
    c.max_step_out = slice.max_step_out;
    c.max_shrink = slice.max_shrink;
    c.w_init = slice.w_init;
    c.save_genes = save_genes;
    c.workers = workers;
    c.sampler_mode = sampler_mode == SamplerMode::conjugate_direct ? CMC_CONJUGATE_DIRECT
                                                                   : CMC_SLICE_FAITHFUL;
    c.concurrent_chains = concurrent_chains ? 1 : 0;
    return c;
  }
};

// Data and model in the reference's row-major layouts (CountMatrix counts
// G x N, ModelSpec X N x L, offsets h, resolved priors).
struct Problem {
  long G = 0, N = 0, L = 0;
  std::vector<long long> counts;
  std::vector<double> X, h;
  double a = 1.0, b = 1.0, d = 1000.0;
  std::vector<double> c, s;  // empty -> reference defaults 10 and 100
  // extension (not in the reference): per-column CMC_PRIOR_* xi priors
  // (empty = the reference's normal prior) and the t prior's k
  std::vector<int> beta_prior;
  double t_df = 1.0;
};

// ChainState (P:include/countmc/types.hpp:86-108) in packed form.
struct ChainState {
  long G = 0, N = 0, L = 0;
  std::vector<double> packed;  // [eps | gamma | beta | theta | sigma | nu | tau]
  double* eps() { return packed.data(); }
  double* gamma() { return eps() + G * N; }
  double* beta() { return gamma() + G; }
  double* theta() { return beta() + G * L; }
  double* sigma() { return theta() + L; }
  double& nu() { return sigma()[L]; }
  double& tau() { return sigma()[L + 1]; }
};

// TuningState (P:include/countmc/engine.hpp:58-74): SliceVar::w / w_aux.
struct TuningState {
  std::vector<double> w, w_aux;
  TuningState() = default;
  // xi_block: G*L with a xi prior (extension; GibbsEngine::tuning_state())
  TuningState(long G, long N, long L, double w_init, long xi_block = 0)
      : w(G * N + G + G * L + L + 2 + xi_block, w_init),
        w_aux(G * N + G + G * L + L + 2 + xi_block, 0.0) {}
};

// ChainOutput (P:include/countmc/engine.hpp:90-108), accumulators in the
// packed order [nu | tau | theta | sigma | beta | gamma | eps].
struct ChainOutput {
  long chain = 0;
  long count = 0;
  std::vector<double> mean, meansq;
  std::vector<double> contrast_prob;
  std::vector<long> contrast_count;
  std::vector<double> samples;  // [column][row]
  std::vector<long> sample_iters;
  std::vector<long> saved_genes;
  std::uint64_t clamp_events = 0;
  ChainState final_state;
};

class GibbsEngine {
 public:
  GibbsEngine(const Problem& p, const RunConfig& cfg,
              const cmc_contrast_set* contrasts = nullptr, int device = 0)
      : G_(p.G), N_(p.N), L_(p.L) {
    std::vector<double> c = p.c.empty() ? std::vector<double>(p.L, 10.0) : p.c;
    std::vector<double> s = p.s.empty() ? std::vector<double>(p.L, 100.0) : p.s;
    cmc_problem cp{p.G, p.N, p.L, p.counts.data(), p.X.data(), p.h.data(),
                   p.a, p.b, p.d, c.data(), s.data(),
                   p.beta_prior.empty() ? nullptr : p.beta_prior.data(), p.t_df};
    for (int v : p.beta_prior) xi_ = xi_ || v != CMC_PRIOR_NORMAL;
    const cmc_run_config cc = cfg.to_c();
    cmc_error e{};
    check(cmc_engine_create(&cp, &cc, contrasts, device, &h_, &e), e);
    cmc_engine_config(h_, &cfg_);
    long n_saved = 0;
    cmc_engine_dims(h_, nullptr, nullptr, nullptr, nullptr, &n_saved, &ncols_, &nrows_);
    saved_.resize(n_saved);
    if (n_saved) cmc_engine_saved_genes(h_, saved_.data());
    n_contrasts_ = contrasts ? contrasts->n_contrasts : 0;
  }
  ~GibbsEngine() { cmc_engine_destroy(h_); }
  GibbsEngine(const GibbsEngine&) = delete;
  GibbsEngine& operator=(const GibbsEngine&) = delete;

  const cmc_run_config& config() const { return cfg_; }
  const std::vector<long>& saved_genes() const { return saved_; }

  // TuningState of this engine's layout at w_init (xi block included)
  TuningState tuning_state() const { return TuningState(G_, N_, L_, cfg_.w_init, XI()); }

  ChainState initial_state(long chain) const {
    ChainState st{G_, N_, L_, std::vector<double>(S())};
    cmc_error e{};
    check(cmc_engine_initial_state(h_, chain, st.packed.data(), &e), e);
    return st;
  }

  // GibbsEngine::iterate: one sweep of `state` in place (device resident
  // during the call); clamps accumulate like ClampCounter.
  void iterate(ChainState& state, TuningState& tuning, long chain, long m,
               std::uint64_t* clamps = nullptr) {
    cmc_error e{};
    check(cmc_engine_set_state(h_, chain, state.packed.data(), tuning.w.data(),
                               tuning.w_aux.data(), &e), e);
    const int rc = cmc_engine_iterate(h_, chain, m, clamps, &e);
    cmc_error e2{};
    check(cmc_engine_get_state(h_, chain, state.packed.data(), tuning.w.data(),
                               tuning.w_aux.data(), &e2), e2);
    check(rc, e);
  }

  // GibbsEngine::run: every chain, batched on the device.
  // write_results (P:src/io.cpp:571-720) for the last run(); labels and ids
  // may be empty ("g<g+1>" / "contrast<k>").
  void write_results(const std::string& outdir, const std::vector<std::string>& genes = {},
                     const std::vector<std::string>& contrast_ids = {},
                     double wall_seconds = 0.0) {
    std::vector<const char*> g, c;
    for (const auto& s : genes) g.push_back(s.c_str());
    for (const auto& s : contrast_ids) c.push_back(s.c_str());
    cmc_error e{};
    check(cmc_engine_write_results(h_, outdir.c_str(), g.empty() ? nullptr : g.data(),
                                   c.empty() ? nullptr : c.data(), wall_seconds, &e),
          e);
  }

  std::vector<ChainOutput> run() {
    cmc_error e{};
    check(cmc_engine_begin(h_, &e), e);
    const long total = cfg_.burnin + cfg_.iterations;
    const long step = progress_ ? 500 : total;
    for (long m = 1; m <= total; m += step) {
      const long m_end = std::min(total + 1, m + step);
      check(cmc_engine_sweeps(h_, m, m_end, &e), e);
      if (progress_) {
        check(cmc_engine_sync(h_, &e), e);
        for (long c = 0; c < cfg_.chains; ++c) progress_(c, m_end - 1, total);
      }
    }
    // the sweeps are enqueued: size (and so page in) the outputs while the
    // device runs, then copy into them after the sync
    std::vector<ChainOutput> outs;
    for (long c = 0; c < cfg_.chains; ++c) outs.push_back(alloc_output(c));
    check(cmc_engine_sync(h_, &e), e);
    for (auto& o : outs) fill_output(o);
    return outs;
  }

  using Progress = std::function<void(long chain, long m, long total)>;
  void set_progress(Progress fn) { progress_ = std::move(fn); }

 private:
  long XI() const { return xi_ ? G_ * L_ : 0; }  // trailing xi block (extension)
  long S() const { return G_ * N_ + G_ + G_ * L_ + 2 * L_ + 2 + XI(); }
  long A() const { return 2 + 2 * L_ + G_ * L_ + G_ + G_ * N_ + XI(); }

  ChainOutput alloc_output(long chain) {
    ChainOutput o;
    o.chain = chain;
    o.mean.resize(A());
    o.meansq.resize(A());
    o.contrast_prob.resize(static_cast<size_t>(G_) * (n_contrasts_ ? n_contrasts_ : 1));
    o.contrast_count.resize(n_contrasts_ ? n_contrasts_ : 1);
    o.samples.resize(static_cast<size_t>(ncols_) * nrows_);
    o.sample_iters.resize(nrows_);
    o.saved_genes = saved_;
    o.final_state = ChainState{G_, N_, L_, std::vector<double>(S())};
    return o;
  }

  void fill_output(ChainOutput& o) {
    cmc_output_view v{};
    v.acc_count = &o.count;
    v.acc_mean = o.mean.data();
    v.acc_meansq = o.meansq.data();
    v.contrast_prob = o.contrast_prob.data();
    v.contrast_count = o.contrast_count.data();
    v.samples = o.samples.data();
    v.sample_iters = o.sample_iters.data();
    v.clamp_events = &o.clamp_events;
    v.final_state = o.final_state.packed.data();
    cmc_error e{};
    check(cmc_engine_get_output(h_, o.chain, &v, &e), e);
  }

  cmc_engine* h_ = nullptr;
  bool xi_ = false;
  cmc_run_config cfg_{};
  long G_, N_, L_;
  long ncols_ = 0, nrows_ = 0;
  int n_contrasts_ = 0;
  std::vector<long> saved_;
  Progress progress_;
};

}  // namespace countmc_b200
