// Internal interface between the engine (engine.cu, which gathers the
// device-resident results) and the host results writer (output_host.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/countmc_b200.h"

namespace cmc {

struct ResultsInput {
  std::string outdir;
  long C = 0, G = 0, N = 0, L = 0;
  const char* const* genes = nullptr;  // G labels; nullptr -> "g<g+1>"
  // per diagnostic row r in [nu, tau, theta L, sigma L, beta G x L, gamma G]
  std::vector<double> rhat, mean, sd, lo, hi;
  std::vector<int> flags;  // bit 0 degenerate, bit 1 pass
  // thinned-sample columns (names in engine order) and their ESS
  std::vector<std::string> col_names;
  std::vector<double> ess;
  std::vector<int> ess_status;  // 0 ok, 1 undefined, 2 degenerate
  std::vector<long> row_col;    // column of each diagnostic row, -1 if not retained
  bool diag_error = false;      // build_diagnostics would throw (C < 2 or M < 2)
  std::string diag_error_msg;
  double z = 0.0;  // normal_quantile(0.975), for the global-contrast intervals
  // contrasts
  std::vector<std::string> contrast_ids;
  std::vector<int> per_gene;
  std::vector<long> prob_off;
  long n_prob = 0;
  std::vector<double> probs;  // [C][n_prob]
  // samples [C][n_cols][rows]
  long rows = 0;
  std::vector<double> samples;
  std::vector<long> sample_iters;
  // run report
  std::string version;
  uint64_t seed = 0;
  long chains = 0, iterations = 0, burnin = 0, tune_cutoff = 0, thin = 0, workers = 0,
       max_step_out = 0, save_genes = 0;
  bool slice_faithful = true;
  double wall_seconds = 0.0;
  std::vector<std::vector<double>> step_seconds;  // [C][7]
  std::vector<uint64_t> clamp_events;             // [C]
  std::vector<long> saved_genes;                  // 0-based
};

// Writes gene_estimates.csv, hyper_estimates.csv, diagnostics.csv,
// samples/chain_<c>.csv and run_report.json like the reference's
// write_results (P:src/io.cpp:571-720).  Returns a CMC_* code.
int write_results_files(const ResultsInput& in, cmc_error* err);

}  // namespace cmc
