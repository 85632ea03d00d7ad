/*
 * countmc_b200.h — C-ABI drop-in boundary for the B200-native Gibbs sweep.
 *
 * This is the boundary a host program links against in place of the
 * reference `countmc::GibbsEngine` (reference: proj/include/countmc/engine.hpp:110-159,
 * implementation proj/src/engine.cpp:42-483).  Plain pointers and sizes
 * only; no C++ or torch types cross it.  Every entry point returns an int
 * status (CMC_OK == 0) and, where it can fail, fills a cmc_error.
 *
 * Packed array layouts (doubles, reference AoS order, so a caller can copy
 * the reference structs in and out with plain memcpy):
 *
 *   state  (S = G*N + G + G*L + 2*L + 2):   [eps G x N | gamma G | beta G x L |
 *                                            theta L | sigma L | nu | tau]
 *       reference ChainState, proj/include/countmc/types.hpp:86-108
 *   tuning (T = G*N + G + G*L + L + 2), one array for SliceVar::w and one for
 *       SliceVar::w_aux:                    [eps G x N | gamma G | beta G x L |
 *                                            sigma L | nu | tau]
 *       reference TuningState, proj/include/countmc/engine.hpp:58-74
 *   accumulators (A = 2 + 2*L + G*L + G + G*N):
 *                                           [nu | tau | theta L | sigma L |
 *                                            beta G x L | gamma G | eps G x N]
 *       reference ChainOutput, proj/include/countmc/engine.hpp:90-108
 */
#ifndef COUNTMC_B200_H
#define COUNTMC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CMC_OK 0
#define CMC_ERR_CONFIG 1 /* reference ConfigError (errors.hpp:10-13)      */
#define CMC_ERR_STALL 2  /* reference SamplerStallError (errors.hpp:36-71) */
#define CMC_ERR_CUDA 3   /* device/runtime failure                         */
#define CMC_ERR_NCCL 4   /* collective failure (multi-GPU)                 */
#define CMC_ERR_ARG 5    /* bad pointer / index at the boundary            */
#define CMC_ERR_LOAD 6   /* reference LoadError (errors.hpp:16-19)         */

/* Sampler modes, reference SamplerMode (engine.hpp:19). */
#define CMC_SLICE_FAITHFUL 0
#define CMC_CONJUGATE_DIRECT 1

/* Contrast parameter families, reference ParamFamily (streaming.hpp:45). */
#define CMC_FAM_BETA_COL 0
#define CMC_FAM_GAMMA 1
#define CMC_FAM_THETA 2
#define CMC_FAM_SIGMA 3
#define CMC_FAM_NU 4
#define CMC_FAM_TAU 5

/* Error record.  For CMC_ERR_STALL the fields mirror SamplerStallError:
 * step in {"epsilon","gamma","nu","tau","beta","sigma"}, 1-based
 * (index1, index2) with -1 where not applicable, the stalled x0, width
 * and iteration; msg is formatted exactly as errors.cpp:8-16 does. */
typedef struct cmc_error {
  int code;
  char step[16];
  long index1;
  long index2;
  long iteration;
  double x0;
  double width;
  char msg[256];
} cmc_error;

/* Data + model.  Replaces CountMatrix (types.hpp:50-60) and ModelSpec
 * (types.hpp:74-83).  counts is G x N row-major (the reference Grid); X is
 * N x L row-major; priors as PriorConfig (types.hpp:62-72), c and s already
 * resolved to length L (PriorConfig::resolve, types.cpp:38-43). */
typedef struct cmc_problem {
  long G;
  long N;
  long L;
  const long long* counts;
  const double* X;
  const double* h;
  double a;
  double b;
  double d;
  const double* c;
  const double* s;
  /* Optional xi-augmented beta priors (SURVEY.md section 8(f) rank 4,
   * BASELINE configs 2-3).  NOT in the reference -- parity unpinned; the
   * parameterisation is DESIGN.md section 7's:
   *   beta_gl ~ N(theta_l, sigma_l^2 xi_gl),  xi_gl ~ prior_l, with
   *   NORMAL xi = 1, LAPLACE xi ~ Exp(rate 1/2), T xi ~ IG(k/2, k/2),
   *   HORSESHOE sqrt(xi) ~ Cauchy+(0, 1).
   * beta_prior: L entries, NULL = all normal (the reference model).
   * t_df: k of the t prior (> 0 when any column is T).  With any non-normal
   * column the packed layouts gain a trailing xi block of G x L entries:
   * state [... | tau | xi], tuning [... | tau | xi], accumulators
   * [... | eps | xi]. */
  const int* beta_prior;
  double t_df;
} cmc_problem;

#define CMC_PRIOR_NORMAL 0
#define CMC_PRIOR_LAPLACE 1
#define CMC_PRIOR_T 2
#define CMC_PRIOR_HORSESHOE 3

/* RunConfig (engine.hpp:21-36) with SliceConfig (slice.hpp:11-17) inlined.
 * tune_cutoff < 0 resolves to min(500, burnin/10) (engine.cpp:33). */
typedef struct cmc_run_config {
  long chains;
  long iterations;
  long burnin;
  long tune_cutoff;
  long thin;
  uint64_t seed;
  int max_step_out;
  int max_shrink;
  double w_init;
  long save_genes;
  int workers;
  int sampler_mode;
  int concurrent_chains;
} cmc_run_config;

/* Flattened ContrastSpec list (streaming.hpp:59-66).  Contrast k owns
 * n_terms[k] consecutive terms; term t owns n_coefs[t] consecutive
 * (family, index, coef) triples and threshold[t].  Scope (per gene vs
 * global) is inferred as ContrastSpec::finalize does (streaming.cpp:76-88). */
typedef struct cmc_contrast_set {
  int n_contrasts;
  const int* n_terms;
  const int* n_coefs;
  const double* threshold;
  const int* family;
  const int* index;
  const double* coef;
} cmc_contrast_set;

/* Destination buffers for one chain's ChainOutput; any pointer may be NULL.
 * Sizes: acc_* [A]; contrast_prob [sum over contrasts of (per_gene ? G : 1)];
 * contrast_count [n_contrasts]; samples [n_cols * n_rows] column-major
 * (samples[col * n_rows + row], reference samples[column][row]);
 * sample_iters [n_rows]; final_state [S]. */
typedef struct cmc_output_view {
  long* acc_count;
  double* acc_mean;
  double* acc_meansq;
  double* acc_mean_c;
  double* acc_meansq_c;
  double* contrast_prob;
  long* contrast_count;
  double* samples;
  long* sample_iters;
  uint64_t* clamp_events;
  double* final_state;
  double* step_seconds; /* [7], the reference StepTimings order (epsilon,
                           gamma, nu, tau, beta, theta, sigma): per-step
                           device seconds after a run in the per-step timing
                           mode (cmc_engine_set_step_timing), else the fused
                           sweep's device time in slot 0 */
} cmc_output_view;

typedef struct cmc_engine cmc_engine;

/* Library identity: returns a static string (build flags, arch). */
const char* cmc_version(void);

/* GibbsEngine::GibbsEngine (engine.cpp:42-91): validates inputs, resolves
 * the config, precomputes A = y X and the column groups, selects saved
 * genes, uploads the SoA problem to `device` and allocates state for all
 * chains.  Rank/world describe gene sharding (1 GPU: rank 0 of 1). */
int cmc_engine_create(const cmc_problem* problem, const cmc_run_config* config,
                      const cmc_contrast_set* contrasts, int device,
                      cmc_engine** out, cmc_error* err);
/* Device buffers come from the device's default memory pool
 * (cudaMallocAsync); on first use of a device the library raises that
 * pool's release threshold to 16 GB (CMC_POOL_RETAIN_MB, 0 = leave the
 * driver default) so later engines reuse freed memory.  Destroy
 * synchronises the device before returning the buffers. */
int cmc_engine_destroy(cmc_engine* engine);

/* Sizes: G, N, L, chains, number of saved genes, thinned columns, rows. */
int cmc_engine_dims(const cmc_engine* engine, long* G, long* N, long* L,
                    long* chains, long* n_saved, long* n_cols, long* n_rows);
/* GibbsEngine::saved_genes (engine.hpp:117), 0-based, ascending. */
int cmc_engine_saved_genes(const cmc_engine* engine, long* out);
/* RunConfig after resolve(): tune_cutoff etc. */
int cmc_engine_config(const cmc_engine* engine, cmc_run_config* out);

/* GibbsEngine::initial_state (engine.cpp:98-142) into a host [S] array. */
int cmc_engine_initial_state(const cmc_engine* engine, long chain,
                             double* state, cmc_error* err);

/* Device-resident state of one chain: upload/download the packed state
 * and tuning (w, w_aux).  Tuning pointers may be NULL on get. */
int cmc_engine_set_state(cmc_engine* engine, long chain, const double* state,
                         const double* tuning_w, const double* tuning_waux,
                         cmc_error* err);
int cmc_engine_get_state(cmc_engine* engine, long chain, double* state,
                         double* tuning_w, double* tuning_waux, cmc_error* err);

/* GibbsEngine::iterate (engine.cpp:161-370): one full sweep at global
 * iteration m (1-based) of the device-resident state of `chain`.  Tuning is
 * active while m <= burnin.  clamps (may be NULL) is incremented by the
 * number of clamp events, as ClampCounter::bump does (model.hpp:18-26). */
int cmc_engine_iterate(cmc_engine* engine, long chain, long m,
                       uint64_t* clamps, cmc_error* err);

/* GibbsEngine::run (engine.cpp:457-483) for every chain: initial state,
 * burn-in + monitored iterations, accumulators, contrasts, thinning.
 * Chains are batched across the grid; the result per chain equals the
 * reference's run_chain(c) (engine.cpp:378-455). */
int cmc_engine_run(cmc_engine* engine, cmc_error* err);

/* The same run split in pieces for benchmarking and progress reporting:
 * begin() loads every chain's initial state and fresh tuning and clears
 * the monitors; sweeps(m_begin, m_end) enqueues iterations
 * m_begin..m_end-1 of run_chain's loop body for all chains on the
 * engine's stream (asynchronous, replayed from a CUDA graph); sync()
 * waits and turns a device stall record into CMC_ERR_STALL. */
int cmc_engine_begin(cmc_engine* engine, cmc_error* err);
int cmc_engine_sweeps(cmc_engine* engine, long m_begin, long m_end,
                      cmc_error* err);
int cmc_engine_sync(cmc_engine* engine, cmc_error* err);
/* Per-step timing mode (debug; reference StepTimings, engine.hpp:86-88 and
 * engine.cpp:173-176): while on, sweeps() launches each step on its own
 * (the gene kernel split into its step-2 and step-5 launches) with CUDA
 * events between them, and get_output()/write_results() report seconds per
 * step; results are bit-identical, the sweep is slower.  Single GPU. */
int cmc_engine_set_step_timing(cmc_engine* engine, int on);
/* Capture (and cache) the CUDA graphs a sweeps() call of `sweeps` sweeps
 * replays, without running them: moves the one-time capture cost out of a
 * timed region.  After begin(); no reference counterpart. */
int cmc_engine_prepare(cmc_engine* engine, long sweeps, cmc_error* err);
/* cudaStream_t the engine launches on (for event timing by the caller). */
void* cmc_engine_stream(cmc_engine* engine);
/* Kernel launches per sweep (gene kernel + hyper tail [+ contrast]). */
int cmc_engine_launches_per_sweep(const cmc_engine* engine);

/* Per-kernel timing of `reps` further monitored sweeps (continuing the
 * run, launched one kernel at a time with CUDA events between them on the
 * engine stream): average device ms of the fused gene-sweep kernel and of
 * the reduction/hyper tail per sweep. */
int cmc_engine_profile(cmc_engine* engine, long m_begin, long reps,
                       double* gene_ms, double* tail_ms, cmc_error* err);
/* The same per sweep phase (single GPU): ms[CMC_PHASES] = average device ms
 * of eps (step 1), gene (steps 2 + 5, and the leaf sums of steps 3/4/6
 * without a xi prior), xi (extension), hyper_a (nu, tau, theta: steps 3, 4,
 * 6; with a xi prior leaf_a, its leaf sums and those draws), leaf_b
 * (reductions + sigma, step 7, and the hyper monitors), gene_contrast;
 * each phase one launch for all chains, phases serialised with CUDA events
 * between them. */
#define CMC_PHASES 6
int cmc_engine_profile_phases(cmc_engine* engine, long m_begin, long reps,
                              double* ms, cmc_error* err);

/* Post-run diagnostics (reference build_diagnostics, src/io.cpp:507-569,
 * over src/diagnostics.cpp), computed on the device from the resident
 * accumulators after run()/sweeps(): one row per parameter in ChainOutput
 * order [nu | tau | theta L | sigma L | beta G x L | gamma G]
 * (R = 2 + 2L + G(L+1) rows): Gelman-Rubin rhat, the pooled mean and sd
 * and the normal-approximation 95% interval (pool_moments /
 * credible_interval); flags bit0 = degenerate (W = 0), bit1 = pass
 * (rhat < 1.1 or degenerate), bit2 = accumulator corruption.  ESS
 * (Geyer initial positive sequence) for every retained thinned column, in
 * sample order; ess_status 0 ok, 1 undefined (< 4 rows), 2 degenerate.
 * Needs >= 2 chains (ConfigError otherwise, as gelman_rhat). */
typedef struct cmc_diag_view {
  double* rhat;
  double* mean;
  double* sd;
  double* ci_lo;
  double* ci_hi;
  int* flags;
  double* ess;
  int* ess_status;
} cmc_diag_view;
int cmc_engine_diagnostics(cmc_engine* engine, const cmc_diag_view* out,
                           cmc_error* err);

/* Profiling aid: warp-level timeline {kernel<<56|slot<<48|smid<<32|block,
 * t_start_ns, t_end_ns} of the next `sweeps` sweeps (direct launches). */
int cmc_engine_trace(cmc_engine* engine, long m_begin, long sweeps,
                     unsigned long long* out, long cap, long* n_out, cmc_error* err);

/* ChainOutput of one chain after run()/sweeps(); see cmc_output_view. */
int cmc_engine_get_output(cmc_engine* engine, long chain,
                          const cmc_output_view* out, cmc_error* err);

/* Synthetic data in the shape of simulate.cpp:28-90 (beta ~ N(theta,
 * sigma^2), gamma ~ IG(nu/2, nu tau/2), eps ~ N(0, gamma), y ~ Poisson):
 * host-side input generator for benchmarks/tests (not on the hot path).
 * counts_out is G x N row-major. */
int cmc_simulate(long G, long N, long L, const double* X, const double* h,
                 double nu, double tau, const double* theta,
                 const double* sigma, uint64_t seed, long long* counts_out,
                 cmc_error* err);

/* Loads one chain's ChainOutput (the layout cmc_engine_get_output fills;
 * every pointer but final_state, contrast_prob, samples and clamp_events is
 * required) into an unsharded engine of the full problem, as if its own
 * run() had produced it: how a sharded job's results, gathered and merged
 * on one rank, reach cmc_engine_diagnostics / cmc_engine_write_results.
 * Every chain must carry the same monitored count.  No reference
 * counterpart (the reference has no sharding). */
int cmc_engine_set_output(cmc_engine* engine, long chain, const cmc_output_view* out,
                          cmc_error* err);

/* Gene sharding (multi-GPU, one process per GPU): restricts the engine to
 * genes [g_begin, g_end) of the full problem (g_begin a multiple of 1024,
 * the reference reduction leaf, parallel.hpp:60) and joins an NCCL clique
 * identified by the 128-byte ncclUniqueId.  Leaf partial sums are
 * all-gathered every sweep, so results are bit-identical for any rank
 * count.  Must be called before begin()/iterate(). */
int cmc_engine_shard(cmc_engine* engine, int rank, int world,
                     const void* nccl_unique_id, cmc_error* err);
/* Writes the 128-byte ncclUniqueId for rank 0 to broadcast. */
int cmc_nccl_unique_id(void* out128, cmc_error* err);
/* Shard bounds for gene count G over `world` ranks (leaf aligned). */
int cmc_shard_bounds(long G, int rank, int world, long* g_begin, long* g_end);

/* Test hook, no reference counterpart: an in-process stand-in for the
 * clique.  `world` engines of one process (one device, one host thread
 * each) join a loopback group in place of cmc_engine_shard and run the
 * sharded path as ranks 0..world-1; the all-gather becomes event-ordered
 * device copies between the engines with a host barrier per exchange.
 * Eager launches and one chain lane only; for parity tests on one GPU. */
typedef struct cmc_loopback cmc_loopback;
int cmc_loopback_create(int world, cmc_loopback** out, cmc_error* err);
int cmc_loopback_destroy(cmc_loopback* group);
int cmc_engine_shard_loopback(cmc_engine* engine, int rank, cmc_loopback* group,
                              cmc_error* err);

/* Results files, replaces countmc::write_results (P:src/io.cpp:571-720):
 * gene_estimates.csv, hyper_estimates.csv, diagnostics.csv,
 * samples/chain_<c>.csv and run_report.json under outdir, from the
 * device-resident accumulators (diagnostics on the device, parallel host
 * formatting).  genes: G labels (NULL -> "g1".."gG", the names generate()
 * gives); contrast_ids: one id per contrast passed to create (NULL ->
 * "contrast<k>").  The CSV bytes equal the reference's for equal inputs.
 * Fewer than 2 chains or 2 monitored iterations: the estimate files are
 * written, then CMC_ERR_CONFIG as build_diagnostics throws. */
int cmc_engine_write_results(cmc_engine* engine, const char* outdir,
                             const char* const* genes,
                             const char* const* contrast_ids,
                             double wall_seconds, cmc_error* err);

/* ---- Input side, host, multithreaded ---- */

/* Parsed counts CSV; replaces countmc::CountMatrix from load_counts
 * (P:src/io.cpp:125-164).  Header "gene,<sample>..." (>= 2 cells, quoted
 * cells per split_csv io.cpp:46-76), one row per gene with N+1 cells, empty
 * rows skipped, CRLF accepted.  Errors are CMC_ERR_LOAD with the
 * reference's LoadError message for the first bad row in file order. */
typedef struct cmc_counts cmc_counts;
int cmc_counts_load(const char* path, cmc_counts** out, cmc_error* err);
int cmc_counts_dims(const cmc_counts* counts, long* G, long* N,
                    int* duplicate_genes);
/* G x N row-major, valid until cmc_counts_free. */
const long long* cmc_counts_data(const cmc_counts* counts);
const char* cmc_counts_gene(const cmc_counts* counts, long g);
const char* cmc_counts_sample(const cmc_counts* counts, long n);
/* All labels at once: which = 0 genes, 1 samples; *blob holds them
 * NUL-terminated back to back (*bytes in total, in row/column order). */
int cmc_counts_labels(const cmc_counts* counts, int which, const char** blob,
                      size_t* bytes);
void cmc_counts_free(cmc_counts* counts);

/* The small input tables of run_fit.  cmc_model_matrix_load replaces
 * load_model_matrix (P:src/io.cpp:178-205): rows = N samples, cols = L,
 * data N x L row-major, names = the header's effect labels.
 * cmc_offsets_load replaces load_offsets (P:src/io.cpp:221-243): rows = N,
 * cols = 1, data = h.  Numbers parse as strtod over the whole cell; errors
 * are CMC_ERR_LOAD with the reference's LoadError messages. */
typedef struct cmc_table cmc_table;
int cmc_model_matrix_load(const char* path, cmc_table** out, cmc_error* err);
int cmc_offsets_load(const char* path, cmc_table** out, cmc_error* err);
int cmc_table_dims(const cmc_table* table, long* rows, long* cols);
const double* cmc_table_data(const cmc_table* table);
const char* cmc_table_name(const cmc_table* table, long col);
void cmc_table_free(cmc_table* table);

/* Median-of-ratios offsets, replaces countmc::estimate_offsets
 * (P:src/model.cpp:21-68; bit-identical).  counts is G x N row-major;
 * h_out has N entries.  No gene positive in every sample -> CMC_ERR_CONFIG
 * with the reference's NormalizationError message. */
int cmc_estimate_offsets(long G, long N, const long long* counts,
                         double* h_out, cmc_error* err);

#ifdef __cplusplus
}
#endif

#endif /* COUNTMC_B200_H */
