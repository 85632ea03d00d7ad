// Device-side data layout of the B200 Gibbs sweep and the launch wrappers
// the host engine (engine.cu) calls.  See DESIGN.md "Data layout in HBM".
//
// Gene state is structure-of-arrays, gene index fastest, so adjacent
// threads (= adjacent genes) touch adjacent 8-byte words:
//   y[n][g], eps[n][g], eps_w[n][g], eps_wa[n][g], gamma[g], beta[l][g],
//   A[l][g], accumulators acc_*[4][k][g] (mean, meansq, mean_c, meansq_c).
// Every per-chain array is repeated with a chain stride; chains are the
// grid's y dimension.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/countmc_b200.h"

namespace cmc {

constexpr int kLMax = 16;         // model-matrix columns supported
constexpr int kLeaf = 1024;       // reference reduction leaf, P:include/countmc/parallel.hpp:60
constexpr int kGeneBlock = 128;   // threads (= genes) per eps / xi block
#ifndef CMC_GENE_THREADS
#define CMC_GENE_THREADS 128
#endif
constexpr int kGeneThreads = CMC_GENE_THREADS;  // threads (= genes) per gene block
constexpr int kTailWarps = 16;    // warps per leaf/hyper block (512 threads)
constexpr int kMaxContrasts = 8;
constexpr int kMaxTerms = 32;
constexpr int kMaxCoefs = 64;
constexpr unsigned long long kNoError = ~0ull;

// Stall key: (step rank 4 bits | column 8 bits | gene 32 bits | sample 20
// bits) so that the numerically smallest key is the stall the reference's
// sequential sweep would hit first (steps 1..7 in order, beta column-major
// over genes, P:src/engine.cpp:178-369).
__host__ __device__ inline unsigned long long stall_key(unsigned step,
                                                        unsigned col,
                                                        unsigned long long g,
                                                        unsigned n) {
  return ((unsigned long long)step << 60) | ((unsigned long long)col << 52) |
         (g << 20) | (unsigned long long)n;
}

// Hyperparameters, their tuning, monitors and bookkeeping for one chain.
struct Hyper {
  double nu, tau;
  double theta[kLMax];
  double sigma[kLMax];
  double w_nu, wa_nu, w_tau, wa_tau;
  double w_sigma[kLMax];
  double wa_sigma[kLMax];
  // Welford monitors [mean, meansq, mean_c, meansq_c] x [nu, tau, theta, sigma]
  double acc[4][2 + 2 * kLMax];
  unsigned long long clamps;
  unsigned long long err_key;
  double err_x0[2 + kLMax];  // nu, tau, sigma_l
  double err_w[2 + kLMax];
  long long err_m;            // iteration of the recorded stall
  unsigned long long err_key_eps;  // stall slot of the eps kernel
  long long err_m_eps;
  unsigned int doneA, doneB;  // last-block counters of the two leaf phases
  // sharded runs: another rank's chain stalled (seen in the gathered stall
  // flags); this rank's kernels of the chain stop, and sync reports the
  // stalling rank's record (exchanged across ranks)
  unsigned int peer_stall;
};

struct ContrastTable {
  int n;
  int gene_needs_hyper;  // a per-gene contrast reads theta/sigma/nu/tau
  int per_gene[kMaxContrasts];
  int term_begin[kMaxContrasts + 1];
  int coef_begin[kMaxTerms + 1];
  double threshold[kMaxTerms];
  int fam[kMaxCoefs];
  int idx[kMaxCoefs];
  double coef[kMaxCoefs];
  long prob_off[kMaxContrasts];
  long n_prob;  // per chain
};

struct SweepParams {
  // problem (this shard)
  int G;         // local genes
  int N, L;
  long g0;       // global index of the first local gene
  long G_total;  // genes over all shards
  int n_leaves_local;
  int n_leaves_total;
  int leaves_per_rank;  // leaf stride of the gathered partial buffers
  int world;
  int Jmax;
  int eps_solo;    // one chain lane: the eps kernel variant tuned to run alone
  int beta_carry;  // gene kernel carries exp(lp_n) across the beta columns (beta_carry_ok)
  int fuse_tail;  // single GPU: the last leaf block runs the hyper step
  int fuse_leaf_a;  // the gene kernel's last block per leaf sums it (no xi prior)
  unsigned int* leaf_cnt;  // [slots][n_leaves_local] finished gene blocks per leaf
  const double* y;  // [N][G]
  const double* A;  // [L][G]
  const double* X;  // [N*L] row-major
  const double* h;  // [N]
  const int* grp_off;   // [L+1]
  const double* grp_val;
  const int* grp_moff;  // [n_groups+1]
  const int* grp_mem;
  double a, b, d;
  double c[kLMax], s[kLMax];
  double exp_clamp;  // exp(700) as the host libm rounds it
  // config
  uint64_t seed;
  int chain_base;  // chain id of grid.y == 0
  int slot_base;   // state slot of grid.y == 0
  int K, max_shrink;
  uint64_t k_reject, k_inv;  // uniform_int(K+1) constants
  long burnin, tune_cutoff, thin, n_rows, n_cols, n_saved;
  int direct;
  const long* d_m;  // device iteration base; kernels use *d_m + m_off
  // state, chain stride = element count of one chain
  double *eps, *eps_w, *eps_wa;
  double *gam, *gam_w, *gam_wa;
  double *beta, *beta_w, *beta_wa;
  double *log_gam, *inv_gam;
  Hyper* hyper;
  // monitoring
  int monitor_enabled;  // run_chain semantics (accumulators/contrasts/thin)
  double *acc_eps, *acc_gam, *acc_beta;
  double* cprob;  // [C][n_prob]
  const ContrastTable* ctab;
  int ctab_n, ctab_gene_in_sweep;
  double* samples;  // [C][n_cols][n_rows]
  const int* saved_slot;  // [G] local: saved index or -1
  // reductions
  // Leaf partials of THIS launch's chains (one lane): [world][C][Q][lpr]
  // and [world][C][L][lpr], indexed by slot - slot_base, so each lane's
  // block is contiguous per rank and one all-gather moves it.
  double* partA;  // quantity stride leaf_qs_a(L, xi_any): Q sums + the stall flag
  double* partB;
  int C;          // chains of this launch's lane (stride of the partial buffers)
  // optional block timeline (debug/profiling): per record {kernel<<56 |
  // slot<<48 | smid<<32 | blockIdx.x, t_start_ns, t_end_ns}
  unsigned long long* trace;
  // per-step timing mode: [slots][4] SM clock cycles of the nu, tau and
  // theta draws inside hyper_a (accumulated; null otherwise)
  unsigned long long* step_cycles;
  unsigned int* trace_n;
  unsigned int trace_cap;
  // launch priorities (host side): the tail and gene kernels are on the
  // critical path, the next sweep's eps kernel is not
  int prio_eps, prio_gene, prio_tail;
  // xi-augmented beta priors (extension, no reference: parity unpinned).
  // With xi_any the leaf buffer partA carries 2 + 2L quantities: [log gamma,
  // 1/gamma, S_l, W_l] with S_l = sum beta_l (normal column) or sum
  // beta_l/xi_l, and W_l = sum 1/xi_l; partB holds sum (beta-theta)^2[/xi].
  int xi_any;
  int xi_trips;       // xi kernel: slice trips before the straggling lanes are parked
  int xi_fam[kLMax];  // CMC_PRIOR_* per column
  double t_df;
  double *xi, *xi_w, *xi_wa;  // [C][L][G]
  double* acc_xi;             // [C][4][L][G]
};

// leaf quantities of partA
__host__ __device__ inline int leaf_q_a(int L, int xi_any) { return 2 + L + (xi_any ? L : 0); }
// quantity stride of partA: the Q sums, then this rank's stall flag of the
// chain at leaf slot 0 (gathered with the sums, read by hyper_a)
__host__ __device__ inline int leaf_qs_a(int L, int xi_any) { return leaf_q_a(L, xi_any) + 1; }
constexpr int kBlocksPerLeaf = kLeaf / kGeneThreads;  // gene blocks per reduction leaf
constexpr int kStage = 128;  // values per warp per staging round of the serial leaf sums
#ifndef CMC_STAGE_EPI
#define CMC_STAGE_EPI 256
#endif
constexpr int kStageEpi = CMC_STAGE_EPI;  // the same in the gene kernel's epilogue (2 x per warp)

// Launch wrappers (sweep_kernels.cu).  `chains` = grid.y.
cudaError_t launch_eps_sweep(const SweepParams& p, int chains, long m_off,
                             cudaStream_t s);
// phase: 3 the whole gene kernel (steps 2 and 5), 1 step 2 only, 2 step 5
// only (the per-step timing mode)
cudaError_t launch_gene_sweep(const SweepParams& p, int chains, long m_off,
                              cudaStream_t s, int phase = 3);
cudaError_t launch_xi_sweep(const SweepParams& p, int chains, long m_off,
                            cudaStream_t s);
cudaError_t launch_leaf_a(const SweepParams& p, int chains, long m_off,
                          cudaStream_t s);
cudaError_t launch_hyper_a(const SweepParams& p, int chains, long m_off,
                           cudaStream_t s);
cudaError_t launch_leaf_b(const SweepParams& p, int chains, long m_off,
                          cudaStream_t s);
cudaError_t launch_hyper_b(const SweepParams& p, int chains, long m_off,
                           cudaStream_t s);
cudaError_t launch_gene_contrast(const SweepParams& p, int chains, long m_off,
                                 cudaStream_t s);
cudaError_t launch_advance(long* d_m, long by, cudaStream_t s);
cudaError_t launch_fill(double* p, size_t n, double v, cudaStream_t s);
cudaError_t launch_fastmath_setup(cudaStream_t s);
cudaError_t launch_compute_A(const double* y, const double* X, double* A,
                             int G, int N, int L, cudaStream_t s);
int gene_sweep_smem_bytes(int N, int Jmax);
// The register-group gene kernel (Jmax <= 2) carries exp(lp_n) through the
// beta columns in a second [N][B] shared array when that keeps it at its
// resident block count (N <= kBetaCarryMaxN; CMC_BETA_CARRY=0 turns it off).
constexpr int kBetaCarryMaxN = 16;
int beta_carry_ok(int N, int Jmax);
// dynamic shared memory of the gene kernel variant an engine launches
int gene_dyn_smem(int N, int Jmax);
// Raise the dynamic shared-memory opt-in of the gene kernel variant for
// (N, Jmax, xi) on the current device (never lowers it: engines of one
// process may share a device); *total = its static + dynamic bytes per
// block, compared by the caller with the device's opt-in limit.
cudaError_t configure_gene_kernels(int N, int Jmax, int xi_any, int* total);
// [K][G] <-> [G][K] (to_aos: SoA -> AoS) on the device
cudaError_t launch_transpose(const double* src, double* dst, long G, int K, bool to_aos,
                             cudaStream_t s);

}  // namespace cmc

namespace cmc {

// Post-run diagnostics (reference build_diagnostics, P:src/io.cpp:507-569,
// over P:src/diagnostics.cpp): rows [nu | tau | theta L | sigma L |
// beta G x L | gamma G] (ChainOutput order), one thread per row.
struct DiagParams {
  int C, L, N;
  long G, M;            // genes, monitored iterations per chain
  long n_cols, n_rows;  // thinned samples per chain: [n_cols][n_rows]
  const Hyper* hyper;   // [C]
  const double* acc_beta;  // [C][4][L][G]
  const double* acc_gam;   // [C][4][G]
  const double* samples;   // [C][n_cols][n_rows]
  double z;             // normal_quantile(0.975) (host libm, as the reference)
  double *rhat, *mean, *sd, *lo, *hi;  // [R]
  int* flags;           // [R] bit0 degenerate, bit1 pass, bit2 corrupt
  double* ess;          // [n_cols]
  int* ess_status;      // [n_cols] 0 ok, 1 undefined, 2 degenerate
};

cudaError_t launch_diagnostics(const DiagParams& d, cudaStream_t s);

}  // namespace cmc
