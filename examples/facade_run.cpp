// C++ caller of the B200 engine through include/countmc_b200.hpp, written
// the way a user of countmc::GibbsEngine writes it.  Deterministic inputs;
// prints one JSON line that tests/test_gpu_facade.py compares with the
// Python mirror on the same inputs.  With an argument, also writes the
// reference's result files there.
#include <cmath>
#include <cstdio>

#include "countmc_b200.hpp"

int main(int argc, char** argv) {
  using namespace countmc_b200;
  Problem p;
  p.G = 300;
  p.N = 16;
  p.L = 5;
  static const double A[4][4] = {{1, 1, -1, 0}, {1, -1, 1, 0}, {1, 1, 1, 1}, {1, 1, 1, -1}};
  static const double blk[4] = {1, 1, -1, -1};
  p.X.assign(p.N * p.L, 0.0);
  for (long n = 0; n < p.N; ++n) {
    for (int l = 0; l < 4; ++l) p.X[n * 5 + l] = A[(n % 16) / 4][l];
    p.X[n * 5 + 4] = blk[n % 4];
  }
  p.h.assign(p.N, 0.0);
  p.counts.resize(p.G * p.N);
  for (long g = 0; g < p.G; ++g)
    for (long n = 0; n < p.N; ++n)
      p.counts[g * p.N + n] = (long long)((g * 7 + n * 13) % 41 + (g % 5) * 3);
  RunConfig cfg;
  cfg.chains = 2;
  cfg.burnin = 40;
  cfg.iterations = 60;
  cfg.thin = 10;
  cfg.seed = 11;
  cfg.save_genes = 6;
  try {
    GibbsEngine eng(p, cfg);
    // one reference-style iterate() on chain 1 from its initial state
    ChainState st = eng.initial_state(1);
    TuningState tu(p.G, p.N, p.L, 1.0);
    std::uint64_t clamps = 0;
    eng.iterate(st, tu, 1, 1, &clamps);
    auto outs = eng.run();
    if (argc > 1) eng.write_results(argv[1]);  // the reference's result files
    double bsum = 0.0;
    for (long i = 2 + 2 * p.L; i < 2 + 2 * p.L + p.G * p.L; ++i) bsum += outs[0].mean[i];
    std::printf("{\"iter_nu\": %.17g, \"iter_eps0\": %.17g, \"nu0\": %.17g, \"nu1\": %.17g, "
                "\"beta_mean_sum\": %.17g, \"count\": %ld}\n",
                st.nu(), st.eps()[0], outs[0].final_state.nu(), outs[1].final_state.nu(),
                bsum, outs[0].count);
  } catch (const std::exception& ex) {
    std::printf("{\"error\": \"%s\"}\n", ex.what());
    return 1;
  }
  return 0;
}
