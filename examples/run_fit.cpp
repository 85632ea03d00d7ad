// The reference CLI's fit flow (P:tools/main.cpp run_fit: load counts and
// model matrix, estimate offsets, run, write results) through the C++ façade
// (include/countmc_b200.hpp), i.e. what a reference user's program looks
// like after the switch.  The manifest JSON is replaced by arguments:
//
//   run_fit counts.csv model_matrix.csv outdir [chains burnin iterations thin seed]
//
// tests/test_gpu_fit.py compares its result files with the reference's own
// pipeline on the same inputs.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "countmc_b200.hpp"

int main(int argc, char** argv) {
  using namespace countmc_b200;
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s counts.csv model_matrix.csv outdir "
                 "[chains burnin iterations thin seed]\n", argv[0]);
    return 1;
  }
  try {
    const CountMatrix m = load_counts(argv[1]);
    const DesignTable d = load_model_matrix(argv[2]);
    if (d.N != m.N) {
      std::fprintf(stderr, "model matrix has %ld rows but counts have %ld samples\n", d.N, m.N);
      return 1;
    }
    Problem p;
    p.G = m.G;
    p.N = m.N;
    p.L = d.L;
    p.counts = m.counts;
    p.X = d.X;
    p.h = estimate_offsets(m);
    RunConfig cfg;
    if (argc > 4) cfg.chains = std::atol(argv[4]);
    if (argc > 5) cfg.burnin = std::atol(argv[5]);
    if (argc > 6) cfg.iterations = std::atol(argv[6]);
    if (argc > 7) cfg.thin = std::atol(argv[7]);
    if (argc > 8) cfg.seed = std::strtoull(argv[8], nullptr, 10);
    GibbsEngine eng(p, cfg);
    const auto t0 = std::chrono::steady_clock::now();
    const auto outs = eng.run();
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    eng.write_results(argv[3], m.genes, {}, wall);
    unsigned long long clamps = 0;
    for (const auto& o : outs) clamps += o.clamp_events;
    std::printf("{\"G\": %ld, \"N\": %ld, \"L\": %ld, \"chains\": %ld, \"wall_seconds\": %.6f, "
                "\"clamp_events\": %llu, \"output\": \"%s\"}\n",
                m.G, m.N, d.L, (long)outs.size(), wall, clamps, argv[3]);
  } catch (const LoadError& e) {
    std::fprintf(stderr, "load error: %s\n", e.what());
    return 1;
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 1;
  } catch (const SamplerStallError& e) {
    std::fprintf(stderr, "sampler stall: %s\n", e.what());
    return 2;
  }
  return 0;
}
