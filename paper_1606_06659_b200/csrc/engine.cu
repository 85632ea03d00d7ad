// Host side of the C-ABI (include/countmc_b200.h): the B200 replacement of
// countmc::GibbsEngine (P:include/countmc/engine.hpp:110-159,
// P:src/engine.cpp:25-483).  Validation, setup (A = yX, column groups,
// saved genes, initial states) and output assembly run here in C++; every
// sweep runs on the device (sweep_kernels.cu), replayed from CUDA graphs,
// with no per-iteration host round trip.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/countmc_b200.h"
#include "output_host.h"
#include "rng.cuh"
#include "sweep.h"

using namespace cmc;

namespace {

// ------------------------------------------------------------ NCCL (dlopen)
typedef struct {
  char internal[128];
} nccl_uid;
typedef void* nccl_comm;
typedef int (*fn_get_uid)(nccl_uid*);
typedef int (*fn_init_rank)(nccl_comm*, int, nccl_uid, int);
typedef int (*fn_all_gather)(const void*, void*, size_t, int, nccl_comm,
                             cudaStream_t);
typedef int (*fn_destroy)(nccl_comm);
typedef int (*fn_comm_split)(nccl_comm, int, int, nccl_comm*, void*);
typedef const char* (*fn_errstr)(int);

struct NcclApi {
  void* lib = nullptr;
  fn_get_uid get_uid = nullptr;
  fn_init_rank init_rank = nullptr;
  fn_all_gather all_gather = nullptr;
  fn_destroy destroy = nullptr;
  fn_comm_split comm_split = nullptr;  // optional (NCCL >= 2.18): per-lane comms
  fn_errstr errstr = nullptr;
  bool load(std::string& why) {
    if (lib) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (lib) break;
    }
    if (!lib) {
      why = "cannot dlopen libnccl.so.2";
      return false;
    }
    get_uid = (fn_get_uid)dlsym(lib, "ncclGetUniqueId");
    init_rank = (fn_init_rank)dlsym(lib, "ncclCommInitRank");
    all_gather = (fn_all_gather)dlsym(lib, "ncclAllGather");
    destroy = (fn_destroy)dlsym(lib, "ncclCommDestroy");
    comm_split = (fn_comm_split)dlsym(lib, "ncclCommSplit");
    errstr = (fn_errstr)dlsym(lib, "ncclGetErrorString");
    if (!get_uid || !init_rank || !all_gather || !destroy) {
      why = "libnccl is missing symbols";
      return false;
    }
    return true;
  }
};
NcclApi g_nccl;
constexpr int kNcclFloat64 = 8;  // ncclDouble

// ---------------------------------------------------------------- errors
void set_err(cmc_error* err, int code, const std::string& msg) {
  if (!err) return;
  std::memset(err, 0, sizeof(*err));
  err->code = code;
  err->index1 = err->index2 = -1;
  std::snprintf(err->msg, sizeof(err->msg), "%s", msg.c_str());
}

// SamplerStallError message, P:src/errors.cpp:8-16.
void set_stall(cmc_error* err, const char* step, long i1, long i2, double x0,
               double w, long m) {
  if (!err) return;
  std::memset(err, 0, sizeof(*err));
  err->code = CMC_ERR_STALL;
  std::snprintf(err->step, sizeof(err->step), "%s", step);
  err->index1 = i1;
  err->index2 = i2;
  err->x0 = x0;
  err->width = w;
  err->iteration = m;
  std::snprintf(err->msg, sizeof(err->msg),
                "slice sampler stalled: step=%s index=(%ld,%ld) x0=%.17g "
                "width=%.17g iteration=%ld",
                step[0] ? step : "?", i1, i2, x0, w, m);
}

#define CUDA_TRY(expr)                                                      \
  do {                                                                      \
    cudaError_t e_ = (expr);                                                \
    if (e_ != cudaSuccess) {                                                \
      set_err(err, CMC_ERR_CUDA,                                            \
              std::string(#expr) + ": " + cudaGetErrorString(e_));          \
      return CMC_ERR_CUDA;                                                  \
    }                                                                       \
  } while (0)

long matrix_rank(std::vector<double> A, long n, long m, double tol) {
  double maxabs = 0.0;
  for (double v : A) maxabs = std::max(maxabs, std::fabs(v));
  if (maxabs == 0.0) return 0;
  const double thresh = tol * maxabs;
  long rank = 0;
  for (long col = 0; col < m && rank < n; ++col) {
    long pivot = rank;
    for (long r = rank + 1; r < n; ++r)
      if (std::fabs(A[r * m + col]) > std::fabs(A[pivot * m + col])) pivot = r;
    if (std::fabs(A[pivot * m + col]) <= thresh) continue;
    if (pivot != rank)
      for (long c = 0; c < m; ++c) std::swap(A[pivot * m + c], A[rank * m + c]);
    for (long r = rank + 1; r < n; ++r) {
      const double f = A[r * m + col] / A[rank * m + col];
      for (long c = col; c < m; ++c) A[r * m + c] -= f * A[rank * m + c];
    }
    ++rank;
  }
  return rank;
}

// Host fork-join over [0, n) in contiguous chunks (setup and transposes
// only; every element is computed independently, so results do not depend
// on the thread count).
template <class F>
void host_parallel_for(long n, F&& body) {
  unsigned hw = std::thread::hardware_concurrency();
  const long nt = std::max<long>(1, std::min<long>(hw ? hw : 1, n / 4096));
  if (nt <= 1) {
    body(0L, n);
    return;
  }
  std::vector<std::thread> th;
  const long chunk = (n + nt - 1) / nt;
  for (long t = 0; t < nt; ++t) {
    const long lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    th.emplace_back([&body, lo, hi] { body(lo, hi); });
  }
  for (auto& x : th) x.join();
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  // From the device's default memory pool (cmc_engine_destroy synchronises
  // the device before any free).  The pool keeps freed memory for the next
  // engine (set_pool_retention), so an engine created after another one of
  // similar size maps no new pages: cudaMalloc of a Paschold-size engine's
  // state took 17-67 ms per create.  The allocation is ordered on this
  // thread's default stream and synchronised here, so every stream may use
  // the buffer at once.
  cudaError_t alloc(size_t count) {
    n = count;
    if (count == 0) return cudaSuccess;
    cudaError_t r = cudaMallocAsync((void**)&p, sizeof(T) * count, cudaStreamPerThread);
    if (r != cudaSuccess) return r;
    return cudaStreamSynchronize(cudaStreamPerThread);
  }
  void free_() {
    if (p) cudaFreeAsync(p, cudaStreamPerThread);
    p = nullptr;
    n = 0;
  }
};

}  // namespace

#ifndef CMC_GRAPH_CHUNK
#define CMC_GRAPH_CHUNK 50  // sweeps per CUDA graph (A/B: 25 0.3551 ms, 50 0.3531, 100 0.3527)
#endif
#ifndef CMC_MAX_LANES
#define CMC_MAX_LANES 2  // chain lanes (r02 A/B with graph upload: 4 lanes 0.3235 vs 0.3273 ms per monitored sweep, but a whole default run() 2.03 vs 1.99 s of sweeps)
#endif

// In-process stand-in for the NCCL clique (test hook): W engines of one
// process share one device, each driven by its own host thread, and play
// ranks 0..W-1 of a sharded job.  The all-gather becomes stream-ordered
// device copies between the engines' partial buffers, sequenced by CUDA
// events and a host barrier -- no kernel waits on another -- so the whole
// sharded path (leaf-aligned shard bounds, g0-offset RNG sites, the
// [world][C][Q][lpr] partial sections, the standalone hyper kernels) runs
// at world > 1 on one GPU.  Eager launches only (events of another
// engine's stream cannot enter a graph capture), one chain lane.
struct cmc_loopback {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  bool broken = false;  // a rank failed or timed out: every barrier fails
  std::vector<const double*> send;
  std::vector<cudaEvent_t> ready, copied;
  std::vector<std::vector<double>> xrec;  // stall records per rank (sync)
  // false if the group is broken or a peer does not arrive within 120 s (a
  // rank that failed elsewhere never reaches its next exchange)
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || broken; }) ||
        gen == g) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    broken = true;
    cv.notify_all();
  }
};

struct cmc_engine {
  // problem (host copy of the full problem)
  long G_total = 0, N = 0, L = 0;
  std::vector<long long> counts;  // G x N
  std::vector<double> X, h, c, s;
  double a = 1, b = 1, d = 1000;
  cmc_run_config cfg{};
  // column groups, P:src/engine.cpp:62-75
  std::vector<int> grp_off, grp_moff, grp_mem;
  std::vector<double> grp_val;
  int Jmax = 1;
  std::vector<long> saved;  // global, ascending
  // xi-augmented beta priors (extension, no reference: parity unpinned)
  std::vector<int> prior;  // L: CMC_PRIOR_*
  bool xi_any = false;
  double t_df = 1.0;
  // contrasts
  ContrastTable ctab{};
  bool has_ctab = false;
  // sharding
  int rank = 0, world = 1;
  long g0 = 0, G = 0;  // local range
  nccl_comm comm = nullptr;
  // one communicator per chain lane (lane 0: comm; others split from it), so
  // the lanes' all-gathers never interleave on one communicator
  nccl_comm lane_comm[4] = {nullptr, nullptr, nullptr, nullptr};
  int split_lanes = 1;      // lanes of a sharded engine
  cmc_loopback* loop = nullptr;  // test hook: in-process exchange instead of NCCL
  cudaEvent_t loop_ready = nullptr, loop_copied = nullptr;
  bool split_tail = false;  // NCCL exchange between the leaf and hyper kernels
  // device
  int device = 0;
  bool dev_ready = false;
  cudaStream_t stream = nullptr;
  cudaStream_t tail_stream = nullptr;  // reduction/hyper tail, overlaps the
                                       // next iteration's eps kernel
  cudaEvent_t ev_gene = nullptr, ev_tail = nullptr;
  // Chain groups ("lanes"): with >= 2 chains the chains are split in two
  // independent groups on separate stream pairs, so one group's
  // latency-bound gene kernel co-runs with the other's eps kernel.
  struct Lane {
    cudaStream_t s = nullptr, t = nullptr;
    cudaEvent_t ev_gene = nullptr, ev_tail = nullptr, ev_join = nullptr;
    int slot0 = 0, chains = 0;
  };
  Lane lanes[4];
  int n_lanes = 1;
  cudaEvent_t ev_fork = nullptr;
  int C = 1;
  DevBuf<double> y, A, Xd, hd, gval;
  DevBuf<int> goff, gmoff, gmem, saved_slot;
  DevBuf<double> eps, eps_w, eps_wa, gam, gam_w, gam_wa, beta, beta_w, beta_wa;
  DevBuf<double> log_gam, inv_gam, acc_eps, acc_gam, acc_beta, cprob, samples;
  DevBuf<double> partA, partB;
  DevBuf<unsigned int> leaf_cnt;  // [slots][local leaves]: gene blocks done per leaf
  DevBuf<double> stall_x;         // sharded sync: [world][C][4] stall records
  cudaEvent_t ev_coll = nullptr;  // last collective enqueued (any lane): one order
  DevBuf<double> xi, xi_w, xi_wa, acc_xi;  // [C][L][G] (acc: [C][4][L][G])
  DevBuf<double> xfer;  // max(N, L) x G: layout transposes for host transfers
  DevBuf<Hyper> hyper;
  DevBuf<ContrastTable> dctab;
  DevBuf<long> d_m;
  long host_m = 1;  // value of *d_m
  SweepParams base{};
  // graph cache: sweeps per graph -> exec (the 50-sweep chunk of a run,
  // plus the lengths of shorter sweep calls and of a run's remainder)
  static constexpr int kGraphSlots = 6;
  cudaGraphExec_t graph[kGraphSlots] = {};
  long graph_len[kGraphSlots] = {};
  long graph_use[kGraphSlots] = {};
  long graph_clock = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool timing_pending = false;
  double sweep_seconds = 0.0;
  // per-step timing mode (cmc_engine_set_step_timing): sweeps launch one
  // step at a time with CUDA events between the steps; per-chain seconds of
  // the reference's 7 steps (StepTimings, P:include/countmc/engine.hpp:86-88)
  bool step_timing = false, step_timed = false;
  std::vector<double> step_sec;           // [C][7]
  DevBuf<unsigned long long> step_cyc;    // [slots][4]
  bool begun = false;
  long n_cols = 0, n_rows = 0;
};

namespace {

int fail_config(cmc_error* err, const std::string& msg) {
  set_err(err, CMC_ERR_CONFIG, msg);
  return CMC_ERR_CONFIG;
}

long prob_len(const cmc_engine* e) { return e->has_ctab ? e->ctab.n_prob : 0; }

// host wall clock for the CMC_PHASE_LOG set-up split (development aid)
static double tnow() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
// The device's default pool keeps up to this many freed bytes instead of
// returning them to the driver at the next synchronisation (once per
// device, never lowered; CMC_POOL_RETAIN_MB overrides, 0 = driver default).
cudaError_t set_pool_retention(int device) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(done.begin(), done.end(), device) != done.end()) return cudaSuccess;
  done.push_back(device);
  const char* v = std::getenv("CMC_POOL_RETAIN_MB");
  const unsigned long long mb = v ? std::strtoull(v, nullptr, 10) : 16384ull;
  if (mb == 0) return cudaSuccess;
  cudaMemPool_t pool;
  cudaError_t r = cudaDeviceGetDefaultMemPool(&pool, device);
  if (r != cudaSuccess) return r;
  unsigned long long cur = 0;
  r = cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &cur);
  if (r != cudaSuccess) return r;
  unsigned long long want = mb << 20;
  if (cur >= want) return cudaSuccess;
  return cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &want);
}

// Allocate and upload this shard's problem and all chain state.
int ensure_device(cmc_engine* e, cmc_error* err) {
  if (e->dev_ready) return CMC_OK;
  const double Q0 = tnow();
  CUDA_TRY(cudaSetDevice(e->device));
  CUDA_TRY(set_pool_retention(e->device));
  CUDA_TRY(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&e->tail_stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&e->ev_gene, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&e->ev_tail, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming));
  e->n_lanes = e->split_tail ? e->split_lanes : (int)std::min<long>(e->C, CMC_MAX_LANES);
  {
    for (int k = 0; k < e->n_lanes; ++k) {
      cmc_engine::Lane& ln = e->lanes[k];
      ln.slot0 = (int)(k * e->C / e->n_lanes);
      ln.chains = (int)((k + 1) * e->C / e->n_lanes) - ln.slot0;
      if (k == 0) {
        ln.s = e->stream;
        ln.t = e->tail_stream;
        ln.ev_gene = e->ev_gene;
        ln.ev_tail = e->ev_tail;
      } else {
        CUDA_TRY(cudaStreamCreateWithFlags(&ln.s, cudaStreamNonBlocking));
        CUDA_TRY(cudaStreamCreateWithFlags(&ln.t, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&ln.ev_gene, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&ln.ev_tail, cudaEventDisableTiming));
      }
      CUDA_TRY(cudaEventCreateWithFlags(&ln.ev_join, cudaEventDisableTiming));
    }
  }
  CUDA_TRY(cudaEventCreate(&e->ev0));
  CUDA_TRY(cudaEventCreate(&e->ev1));
  const long G = e->G, N = e->N, L = e->L, C = e->C;
  const int Qs = leaf_qs_a((int)L, e->xi_any ? 1 : 0);
  {
    // dynamic shared memory opt-in of the gene kernels on this device; the
    // static part counts against the same per-block limit
    int total = 0, optin = 0;
    CUDA_TRY(configure_gene_kernels((int)N, e->Jmax, e->xi_any ? 1 : 0, &total));
    CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device));
    if (total > optin) {
      set_err(err, CMC_ERR_CONFIG,
              "N (plus 2x the groups per model-matrix column) too large for this build's gene "
              "kernel shared memory");
      return CMC_ERR_CONFIG;
    }
  }
  // SoA y[n][g] as double (exact for counts < 2^53)
  const double Q1 = tnow();
  std::vector<double> yh((size_t)N * G);
  for (long g = 0; g < G; ++g)
    for (long n = 0; n < N; ++n)
      yh[(size_t)n * G + g] = (double)e->counts[(size_t)(e->g0 + g) * N + n];
  CUDA_TRY(e->y.alloc(yh.size()));
  CUDA_TRY(cudaMemcpy(e->y.p, yh.data(), sizeof(double) * yh.size(),
                      cudaMemcpyHostToDevice));
  CUDA_TRY(e->Xd.alloc(e->X.size()));
  CUDA_TRY(cudaMemcpy(e->Xd.p, e->X.data(), sizeof(double) * e->X.size(),
                      cudaMemcpyHostToDevice));
  CUDA_TRY(e->hd.alloc(e->h.size()));
  CUDA_TRY(cudaMemcpy(e->hd.p, e->h.data(), sizeof(double) * e->h.size(),
                      cudaMemcpyHostToDevice));
  CUDA_TRY(e->A.alloc((size_t)L * G));
  CUDA_TRY(launch_compute_A(e->y.p, e->Xd.p, e->A.p, (int)G, (int)N, (int)L,
                            e->stream));
  CUDA_TRY(launch_fastmath_setup(e->stream));
  CUDA_TRY(e->goff.alloc(e->grp_off.size()));
  CUDA_TRY(cudaMemcpy(e->goff.p, e->grp_off.data(), sizeof(int) * e->grp_off.size(),
                      cudaMemcpyHostToDevice));
  CUDA_TRY(e->gmoff.alloc(e->grp_moff.size()));
  CUDA_TRY(cudaMemcpy(e->gmoff.p, e->grp_moff.data(),
                      sizeof(int) * e->grp_moff.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(e->gmem.alloc(std::max<size_t>(1, e->grp_mem.size())));
  if (!e->grp_mem.empty())
    CUDA_TRY(cudaMemcpy(e->gmem.p, e->grp_mem.data(),
                        sizeof(int) * e->grp_mem.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(e->gval.alloc(std::max<size_t>(1, e->grp_val.size())));
  if (!e->grp_val.empty())
    CUDA_TRY(cudaMemcpy(e->gval.p, e->grp_val.data(),
                        sizeof(double) * e->grp_val.size(), cudaMemcpyHostToDevice));
  std::vector<int> slot((size_t)G, -1);
  for (size_t k = 0; k < e->saved.size(); ++k) {
    const long g = e->saved[k] - e->g0;
    if (g >= 0 && g < G) slot[(size_t)g] = (int)k;
  }
  CUDA_TRY(e->saved_slot.alloc(slot.size()));
  CUDA_TRY(cudaMemcpy(e->saved_slot.p, slot.data(), sizeof(int) * slot.size(),
                      cudaMemcpyHostToDevice));
  // chain state: slots 0..C-1 are run()'s chains; slot C is iterate()'s
  // scratch (the reference's iterate works on caller-owned state, so it must
  // not disturb a run).  Accumulators exist for run chains only: iterate()
  // sweeps with the monitors off.
  const double Q2 = tnow();
  const long Cs = C + 1;
  const size_t gn = (size_t)G * N * C, gl = (size_t)G * L * C, gc = (size_t)G * C;
  const size_t sn = (size_t)G * N * Cs, sl = (size_t)G * L * Cs, sc = (size_t)G * Cs;
  CUDA_TRY(e->eps.alloc(sn));
  CUDA_TRY(e->eps_w.alloc(sn));
  CUDA_TRY(e->eps_wa.alloc(sn));
  CUDA_TRY(e->gam.alloc(sc));
  CUDA_TRY(e->gam_w.alloc(sc));
  CUDA_TRY(e->gam_wa.alloc(sc));
  CUDA_TRY(e->beta.alloc(sl));
  CUDA_TRY(e->beta_w.alloc(sl));
  CUDA_TRY(e->beta_wa.alloc(sl));
  CUDA_TRY(e->log_gam.alloc(sc));
  CUDA_TRY(e->inv_gam.alloc(sc));
  CUDA_TRY(e->acc_eps.alloc(4 * gn));
  CUDA_TRY(e->acc_gam.alloc(4 * gc));
  CUDA_TRY(e->acc_beta.alloc(4 * gl));
  if (e->xi_any) {
    CUDA_TRY(e->xi.alloc(sl));
    CUDA_TRY(e->xi_w.alloc(sl));
    CUDA_TRY(e->xi_wa.alloc(sl));
    CUDA_TRY(e->acc_xi.alloc(4 * gl));
  }
  CUDA_TRY(e->cprob.alloc(std::max<long>(1, prob_len(e)) * C));
  CUDA_TRY(e->samples.alloc(std::max<long>(1, e->n_cols * e->n_rows) * C));
  CUDA_TRY(e->hyper.alloc((size_t)Cs));
  CUDA_TRY(cudaMemset(e->hyper.p, 0, sizeof(Hyper) * Cs));
  CUDA_TRY(e->xfer.alloc((size_t)std::max(N, L) * G));
  const long n_leaves_total = (e->G_total + kLeaf - 1) / kLeaf;
  const long lpr = (n_leaves_total + e->world - 1) / e->world;
  CUDA_TRY(e->partA.alloc((size_t)e->world * Cs * Qs * lpr));
  CUDA_TRY(cudaMemset(e->partA.p, 0, sizeof(double) * e->partA.n));
  const long n_leaves_local = (G + kLeaf - 1) / kLeaf;
  CUDA_TRY(e->leaf_cnt.alloc((size_t)Cs * n_leaves_local));
  CUDA_TRY(cudaMemset(e->leaf_cnt.p, 0, sizeof(unsigned int) * e->leaf_cnt.n));
  CUDA_TRY(e->step_cyc.alloc((size_t)Cs * 4));
  CUDA_TRY(cudaMemset(e->step_cyc.p, 0, sizeof(unsigned long long) * e->step_cyc.n));
  if (e->split_tail) CUDA_TRY(e->stall_x.alloc((size_t)e->world * Cs * 4));
  CUDA_TRY(cudaEventCreateWithFlags(&e->ev_coll, cudaEventDisableTiming));
  CUDA_TRY(e->partB.alloc((size_t)e->world * Cs * L * lpr));
  CUDA_TRY(e->dctab.alloc(1));
  CUDA_TRY(cudaMemcpy(e->dctab.p, &e->ctab, sizeof(ContrastTable),
                      cudaMemcpyHostToDevice));
  CUDA_TRY(e->d_m.alloc(1));
  long one = 1;
  CUDA_TRY(cudaMemcpy(e->d_m.p, &one, sizeof(long), cudaMemcpyHostToDevice));
  e->host_m = 1;

  if (std::getenv("CMC_PHASE_LOG"))
    fprintf(stderr, "ensure: streams %.1f ms, inputs %.1f ms, state allocs %.1f ms\n",
            1e3 * (Q1 - Q0), 1e3 * (Q2 - Q1), 1e3 * (tnow() - Q2));
  SweepParams& p = e->base;
  std::memset(&p, 0, sizeof(p));
  p.G = (int)G;
  p.N = (int)N;
  p.L = (int)L;
  p.g0 = e->g0;
  p.G_total = e->G_total;
  p.n_leaves_local = (int)((G + kLeaf - 1) / kLeaf);
  p.n_leaves_total = (int)n_leaves_total;
  p.leaves_per_rank = (int)lpr;
  p.world = e->world;
  p.Jmax = e->Jmax;
  p.beta_carry = beta_carry_ok((int)e->N, e->Jmax);
  p.eps_solo = e->n_lanes == 1 ? 1 : 0;
  p.fuse_tail = e->split_tail ? 0 : 1;
  // without a xi prior the gene kernel sums its own leaves (the xi sums
  // need the xi kernel's draws: leaf_a kernel)
  p.fuse_leaf_a = e->xi_any ? 0 : 1;
  p.leaf_cnt = e->leaf_cnt.p;
  p.y = e->y.p;
  p.A = e->A.p;
  p.X = e->Xd.p;
  p.h = e->hd.p;
  p.grp_off = e->goff.p;
  p.grp_val = e->gval.p;
  p.grp_moff = e->gmoff.p;
  p.grp_mem = e->gmem.p;
  p.a = e->a;
  p.b = e->b;
  p.d = e->d;
  for (long l = 0; l < L; ++l) {
    p.c[l] = e->c[l];
    p.s[l] = e->s[l];
  }
  p.exp_clamp = std::exp(700.0);
  p.seed = e->cfg.seed;
  p.K = e->cfg.max_step_out;
  p.max_shrink = e->cfg.max_shrink;
  {
    const uint64_t n = (uint64_t)e->cfg.max_step_out + 1;
    p.k_reject = (0ull - n) % n;
    p.k_inv = (uint64_t)(((unsigned __int128)1 << 64) / n);
  }
  p.burnin = e->cfg.burnin;
  p.tune_cutoff = e->cfg.tune_cutoff;
  p.thin = e->cfg.thin;
  p.n_rows = e->n_rows;
  p.n_cols = e->n_cols;
  p.n_saved = (long)e->saved.size();
  p.direct = e->cfg.sampler_mode == CMC_CONJUGATE_DIRECT;
  p.d_m = e->d_m.p;
  p.eps = e->eps.p;
  p.eps_w = e->eps_w.p;
  p.eps_wa = e->eps_wa.p;
  p.gam = e->gam.p;
  p.gam_w = e->gam_w.p;
  p.gam_wa = e->gam_wa.p;
  p.beta = e->beta.p;
  p.beta_w = e->beta_w.p;
  p.beta_wa = e->beta_wa.p;
  p.log_gam = e->log_gam.p;
  p.inv_gam = e->inv_gam.p;
  p.hyper = e->hyper.p;
  p.acc_eps = e->acc_eps.p;
  p.acc_gam = e->acc_gam.p;
  p.acc_beta = e->acc_beta.p;
  p.cprob = e->cprob.p;
  p.ctab = e->dctab.p;
  p.ctab_n = e->has_ctab ? e->ctab.n : 0;
  p.ctab_gene_in_sweep = e->has_ctab && !e->ctab.gene_needs_hyper;
  p.samples = e->samples.p;
  p.saved_slot = e->saved_slot.p;
  p.partA = e->partA.p;
  p.partB = e->partB.p;
  p.C = (int)C;
  p.xi_any = e->xi_any ? 1 : 0;
  {
    const char* v = std::getenv("CMC_XI_TRIPS");  // development override (A/B)
    // horseshoe A/B, ms per 4-chain sweep on the final build (two reps):
    // 8 0.767, 10 0.746, 12 0.729, 14 0.732, 16 0.739, 20 0.750, 24 0.760
    // (before the per-model block counts: 8 0.749, 16 0.756, 32 0.787, no
    // parking 0.830)
    p.xi_trips = v ? std::atoi(v) : 12;
  }
  for (long l = 0; l < L; ++l) p.xi_fam[l] = e->prior[(size_t)l];
  p.t_df = e->t_df;
  p.xi = e->xi.p;
  p.xi_w = e->xi_w.p;
  p.xi_wa = e->xi_wa.p;
  p.acc_xi = e->acc_xi.p;
  {
    int least = 0, greatest = 0;
    CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    // the tail and the gene kernel ahead of the eps kernel.  Round 1 (A/B on
    // B200): tail > gene > eps 0.3580 ms/sweep, tail > gene = eps 0.3541,
    // all equal 0.3620, tail > eps > gene 0.3508 vs 0.3507 level; the tail
    // first with gene = eps was kept.  Re-measured on the final round-2
    // build (100-sweep calls, two reps each, scripts/ab_e2e.sh): tail first
    // with gene = eps 0.3260, tail > eps > gene 0.3261, tail > gene > eps
    // 0.3224, tail = gene > eps 0.3214 ms; run() 1.981-1.988 s vs
    // 1.991-1.998 s.  Later: gene > tail > eps 0.3191 vs 0.3193 (level);
    // gene first with the tail last 0.3540 (the tail must not wait).
    // Modes 5 and 6 are those two.
#ifndef CMC_PRIO_MODE
#define CMC_PRIO_MODE 4  // A/B: 0 tail first, eps = gene; 1 all level; 2 tail > eps > gene; 3 tail > gene > eps; 4 tail = gene > eps; 5 gene > tail > eps; 6 gene > eps = tail
#endif
    // With a t or Laplace prior (the plain xi kernel after the gene kernel,
    // at the gene kernel's priority) the gene kernel stays level with eps:
    // t 0.5347 vs 0.5572, Laplace 0.4554 vs 0.4654 ms; the horseshoe (parked
    // xi kernel) follows the normal model: 0.6951 vs 0.7249 ms.
    bool hs = false;
    for (int v : e->prior) hs |= v == CMC_PRIOR_HORSESHOE;
    const int mode = (CMC_PRIO_MODE >= 4 && e->xi_any && !hs) ? 0 : CMC_PRIO_MODE;
    const int mid = (least + greatest) / 2;
    p.prio_eps = least;
    p.prio_tail = mode == 1 ? least : greatest;
    p.prio_gene = least;
    if (mode == 2) p.prio_eps = mid;
    if (mode == 3) p.prio_gene = mid;
    if (mode == 4) p.prio_gene = greatest;
    if (mode == 5) { p.prio_gene = greatest; p.prio_tail = mid; }
    if (mode == 6) { p.prio_gene = greatest; p.prio_tail = least; }
  }
  CUDA_TRY(cudaStreamSynchronize(e->stream));
  e->dev_ready = true;
  return CMC_OK;
}

// GibbsEngine::initial_state, P:src/engine.cpp:98-142 (host, glibc libm:
// bit-identical to the reference on the same machine).
void initial_state_host(const cmc_engine* e, long chain, double* st) {
  const long G = e->G_total, N = e->N, L = e->L;
  double* eps = st;
  double* gam = eps + G * N;
  double* beta = gam + G;
  double* theta = beta + G * L;
  double* sigma = theta + L;
  std::fill(eps, eps + G * N, 0.0);
  std::fill(gam, gam + G, 1.0);
  std::fill(beta, beta + G * L, 0.0);
  std::fill(theta, theta + L, 0.0);
  std::fill(sigma, sigma + L, 1.0);
  double& nu = sigma[L];
  double& tau = sigma[L + 1];
  nu = 2.0;
  tau = 1.0;
  double hbar = 0.0;
  for (double v : e->h) hbar += v;
  hbar /= (double)N;
  host_parallel_for(G, [&](long g0, long g1) {
    for (long g = g0; g < g1; ++g) {
      double mean = 0.0;
      for (long n = 0; n < N; ++n) mean += (double)e->counts[(size_t)g * N + n];
      mean /= (double)N;
      beta[g * L] = std::log(mean + 1.0) - hbar;
    }
  });
  double tbar = 0.0;
  for (long g = 0; g < G; ++g) tbar += beta[g * L];
  theta[0] = tbar / (double)G;
  if (chain > 0) {
    const uint64_t seed = e->cfg.seed, ch = (uint64_t)chain;
    auto z = [&](uint64_t fam, uint64_t flat) {
      Stream s;
      s.init(seed, ch, 0, site_id(fam, flat));
      return 0.5 * normal(s);
    };
    auto clamp_interior = [](double v, double lo, double hi) {
      return std::min(std::max(v, lo), hi);
    };
    host_parallel_for(G, [&](long g0, long g1) {
      for (long g = g0; g < g1; ++g) {
        for (long n = 0; n < N; ++n) eps[g * N + n] += z(kSiteEps, (uint64_t)(g * N + n));
        gam[g] = std::max(1e-3, gam[g] + z(kSiteGamma, (uint64_t)g));
        for (long l = 0; l < L; ++l) beta[g * L + l] += z(kSiteBeta, (uint64_t)(g * L + l));
      }
    });
    for (long l = 0; l < L; ++l) {
      theta[l] += z(kSiteTheta, (uint64_t)l);
      const double sv = e->s[l];
      sigma[l] = clamp_interior(sigma[l] + z(kSiteSigma, (uint64_t)l), 1e-6 * sv,
                                (1.0 - 1e-6) * sv);
    }
    nu = clamp_interior(nu + z(kSiteNu, 0), 1e-6 * e->d, (1.0 - 1e-6) * e->d);
    tau = std::max(1e-3, tau + z(kSiteTau, 0));
  }
  if (e->xi_any) std::fill(sigma + L + 2, sigma + L + 2 + G * L, 1.0);  // xi block
}

// Host AoS block [G_local][K] (the reference's row-major layout) <-> device
// SoA [K][G_local]: one contiguous copy plus a device transpose through
// e->xfer, ordered on the engine stream (the caller synchronises).
cudaError_t aos_to_device(cmc_engine* e, const double* src_aos, double* dst_soa, long K) {
  const long G = e->G;
  cudaError_t r = cudaMemcpyAsync(e->xfer.p, src_aos, sizeof(double) * K * G,
                                  cudaMemcpyHostToDevice, e->stream);
  if (r != cudaSuccess) return r;
  return launch_transpose(e->xfer.p, dst_soa, G, (int)K, false, e->stream);
}
cudaError_t device_to_aos(cmc_engine* e, const double* src_soa, double* dst_aos, long K) {
  const long G = e->G;
  cudaError_t r = launch_transpose(src_soa, e->xfer.p, G, (int)K, true, e->stream);
  if (r != cudaSuccess) return r;
  r = cudaMemcpyAsync(dst_aos, e->xfer.p, sizeof(double) * K * G, cudaMemcpyDeviceToHost,
                      e->stream);
  if (r != cudaSuccess) return r;
  return cudaStreamSynchronize(e->stream);  // the staging buffer is reused next
}

// Upload one chain's packed state (+ optional tuning) into slot `c`.
int upload_state(cmc_engine* e, long c, const double* st, const double* tw,
                 const double* ta, cmc_error* err) {
  const long Gt = e->G_total, G = e->G, N = e->N, L = e->L, g0 = e->g0;
  const double* eps = st;
  const double* gam = eps + Gt * N;
  const double* beta = gam + Gt;
  const double* theta = beta + Gt * L;
  const double* sigma = theta + L;
  std::vector<double> buf((size_t)std::max(N, L) * G);
  auto put_gn = [&](const double* src, double* dst, long K) -> cudaError_t {
    cudaError_t r = aos_to_device(e, src + g0 * K, dst, K);
    if (r != cudaSuccess) return r;
    return cudaStreamSynchronize(e->stream);  // e->xfer is reused by the next call
  };
  const size_t so = (size_t)c;
  CUDA_TRY(put_gn(eps, e->eps.p + so * N * G, N));
  CUDA_TRY(cudaMemcpy(e->gam.p + so * G, gam + g0, sizeof(double) * G,
                      cudaMemcpyHostToDevice));
  {  // 1/gamma, read by the eps kernel (0.5 * inv_gam = 1/(2 gamma))
    host_parallel_for(G, [&](long a, long b) {
      for (long g = a; g < b; ++g) buf[(size_t)g] = 1.0 / gam[g0 + g];
    });
    CUDA_TRY(cudaMemcpy(e->inv_gam.p + so * G, buf.data(), sizeof(double) * G,
                        cudaMemcpyHostToDevice));
  }
  CUDA_TRY(put_gn(beta, e->beta.p + so * L * G, L));
  if (e->xi_any) CUDA_TRY(put_gn(sigma + L + 2, e->xi.p + so * L * G, L));
  if (tw && ta) {
    const double* tws[2] = {tw, ta};
    double* de[2] = {e->eps_w.p, e->eps_wa.p};
    double* dg[2] = {e->gam_w.p, e->gam_wa.p};
    double* db[2] = {e->beta_w.p, e->beta_wa.p};
    for (int k = 0; k < 2; ++k) {
      const double* t = tws[k];
      CUDA_TRY(put_gn(t, de[k] + so * N * G, N));
      CUDA_TRY(cudaMemcpy(dg[k] + so * G, t + Gt * N + g0, sizeof(double) * G,
                          cudaMemcpyHostToDevice));
      CUDA_TRY(put_gn(t + Gt * N + Gt, db[k] + so * L * G, L));
      if (e->xi_any) {
        double* dx = k == 0 ? e->xi_w.p : e->xi_wa.p;
        CUDA_TRY(put_gn(t + Gt * N + Gt + Gt * L + L + 2, dx + so * L * G, L));
      }
    }
  }
  Hyper hp;
  CUDA_TRY(cudaMemcpy(&hp, e->hyper.p + c, sizeof(Hyper), cudaMemcpyDeviceToHost));
  hp.nu = sigma[L];
  hp.tau = sigma[L + 1];
  for (long l = 0; l < L; ++l) {
    hp.theta[l] = theta[l];
    hp.sigma[l] = sigma[l];
  }
  if (tw && ta) {
    const long off = Gt * N + Gt + Gt * L;
    for (long l = 0; l < L; ++l) {
      hp.w_sigma[l] = tw[off + l];
      hp.wa_sigma[l] = ta[off + l];
    }
    hp.w_nu = tw[off + L];
    hp.wa_nu = ta[off + L];
    hp.w_tau = tw[off + L + 1];
    hp.wa_tau = ta[off + L + 1];
  }
  hp.err_key = kNoError;
  hp.err_key_eps = kNoError;
  hp.doneA = hp.doneB = 0;
  hp.peer_stall = 0;
  CUDA_TRY(cudaMemcpy(e->hyper.p + c, &hp, sizeof(Hyper), cudaMemcpyHostToDevice));
  // the per-leaf block counters of this slot (a stalled sweep may have left
  // them mid-count)
  const size_t nl = (size_t)((e->G + kLeaf - 1) / kLeaf);
  CUDA_TRY(cudaMemset(e->leaf_cnt.p + (size_t)c * nl, 0, sizeof(unsigned int) * nl));
  return CMC_OK;
}

int download_state(cmc_engine* e, long c, double* st, double* tw, double* ta,
                   cmc_error* err) {
  const long Gt = e->G_total, G = e->G, N = e->N, L = e->L, g0 = e->g0;
  auto get_gn = [&](const double* src, double* dst, long K) -> cudaError_t {
    return device_to_aos(e, src, dst + g0 * K, K);
  };
  const size_t so = (size_t)c;
  Hyper hp;
  CUDA_TRY(cudaMemcpy(&hp, e->hyper.p + c, sizeof(Hyper), cudaMemcpyDeviceToHost));
  if (st) {
    double* eps = st;
    double* gam = eps + Gt * N;
    double* beta = gam + Gt;
    double* theta = beta + Gt * L;
    double* sigma = theta + L;
    CUDA_TRY(get_gn(e->eps.p + so * N * G, eps, N));
    CUDA_TRY(cudaMemcpy(gam + g0, e->gam.p + so * G, sizeof(double) * G,
                        cudaMemcpyDeviceToHost));
    CUDA_TRY(get_gn(e->beta.p + so * L * G, beta, L));
    for (long l = 0; l < L; ++l) {
      theta[l] = hp.theta[l];
      sigma[l] = hp.sigma[l];
    }
    sigma[L] = hp.nu;
    sigma[L + 1] = hp.tau;
    if (e->xi_any) CUDA_TRY(get_gn(e->xi.p + so * L * G, sigma + L + 2, L));
  }
  double* tws[2] = {tw, ta};
  double* de[2] = {e->eps_w.p, e->eps_wa.p};
  double* dg[2] = {e->gam_w.p, e->gam_wa.p};
  double* db[2] = {e->beta_w.p, e->beta_wa.p};
  for (int k = 0; k < 2; ++k) {
    double* t = tws[k];
    if (!t) continue;
    CUDA_TRY(get_gn(de[k] + so * N * G, t, N));
    CUDA_TRY(cudaMemcpy(t + Gt * N + g0, dg[k] + so * G, sizeof(double) * G,
                        cudaMemcpyDeviceToHost));
    CUDA_TRY(get_gn(db[k] + so * L * G, t + Gt * N + Gt, L));
    const long off = Gt * N + Gt + Gt * L;
    for (long l = 0; l < L; ++l) t[off + l] = k == 0 ? hp.w_sigma[l] : hp.wa_sigma[l];
    t[off + L] = k == 0 ? hp.w_nu : hp.wa_nu;
    t[off + L + 1] = k == 0 ? hp.w_tau : hp.wa_tau;
    if (e->xi_any)
      CUDA_TRY(get_gn(k == 0 ? e->xi_w.p + so * L * G : e->xi_wa.p + so * L * G,
                      t + off + L + 2, L));
  }
  return CMC_OK;
}

// One chain's stall record on the host: iteration (-1: none), packed key
// (sweep.h stall_key, global gene index), stalled value and width.
struct StallRec {
  long long m = -1;
  unsigned long long key = kNoError;
  double x0 = 0.0, w = 0.0;
};

// Decode slot c's device stall record (two slots, see sweep_kernels.cu
// record_stall: the earlier iteration wins, then the smaller key, i.e. the
// reference's sequential order).  A stalled step leaves its value and
// width untouched on the device, where they are read back.
cudaError_t local_stall(cmc_engine* e, long c, StallRec* out) {
  Hyper hp;
  cudaError_t r = cudaMemcpy(&hp, e->hyper.p + c, sizeof(Hyper), cudaMemcpyDeviceToHost);
  if (r != cudaSuccess) return r;
  *out = StallRec{};
  if (hp.err_key == kNoError && hp.err_key_eps == kNoError) return cudaSuccess;
  unsigned long long key = hp.err_key;
  long long km = hp.err_m;
  if (hp.err_key_eps != kNoError &&
      (hp.err_key == kNoError || hp.err_m_eps < hp.err_m ||
       (hp.err_m_eps == hp.err_m && hp.err_key_eps < hp.err_key))) {
    key = hp.err_key_eps;
    km = hp.err_m_eps;
  }
  const unsigned step = (unsigned)(key >> 60);
  const long col = (long)((key >> 52) & 0xff);
  const long g = (long)((key >> 20) & 0xffffffffull);
  const long n = (long)(key & 0xfffff);
  double x0 = 0, w = 0;
  if (step == 1 || step == 2 || step == 5) {
    const size_t gl = (size_t)(g - e->g0), G = (size_t)e->G;
    // step 5 with n == 1 is xi_gl (extension), drawn right after beta_gl
    const bool xs5 = step == 5 && n == 1;
    const double* xs = step == 1 ? e->eps.p + (size_t)c * e->N * G + (size_t)n * G + gl
                       : step == 2 ? e->gam.p + (size_t)c * G + gl
                       : xs5       ? e->xi.p + (size_t)c * e->L * G + (size_t)col * G + gl
                                   : e->beta.p + (size_t)c * e->L * G + (size_t)col * G + gl;
    const double* ws = step == 1 ? e->eps_w.p + (size_t)c * e->N * G + (size_t)n * G + gl
                       : step == 2 ? e->gam_w.p + (size_t)c * G + gl
                       : xs5       ? e->xi_w.p + (size_t)c * e->L * G + (size_t)col * G + gl
                                   : e->beta_w.p + (size_t)c * e->L * G + (size_t)col * G + gl;
    if ((r = cudaMemcpy(&x0, xs, sizeof(double), cudaMemcpyDeviceToHost)) != cudaSuccess) return r;
    if ((r = cudaMemcpy(&w, ws, sizeof(double), cudaMemcpyDeviceToHost)) != cudaSuccess) return r;
  } else {
    const int k = step == 3 ? 0 : step == 4 ? 1 : 2 + (int)col;
    x0 = hp.err_x0[k];
    w = hp.err_w[k];
  }
  *out = StallRec{km, key, x0, w};
  return cudaSuccess;
}

void report_stall(const StallRec& s, cmc_error* err) {
  const unsigned step = (unsigned)(s.key >> 60);
  const long col = (long)((s.key >> 52) & 0xff);
  const long g = (long)((s.key >> 20) & 0xffffffffull);
  const long n = (long)(s.key & 0xfffff);
  const long it = (long)s.m;
  switch (step) {
    case 1: set_stall(err, "epsilon", g + 1, n + 1, s.x0, s.w, it); break;
    case 2: set_stall(err, "gamma", g + 1, -1, s.x0, s.w, it); break;
    case 3: set_stall(err, "nu", -1, -1, s.x0, s.w, it); break;
    case 4: set_stall(err, "tau", -1, -1, s.x0, s.w, it); break;
    case 5: set_stall(err, n == 1 ? "xi" : "beta", g + 1, col + 1, s.x0, s.w, it); break;
    default: set_stall(err, "sigma", col + 1, -1, s.x0, s.w, it); break;
  }
}

// Sharded runs: every rank's records of slots [lo, hi) to every rank, so
// all ranks raise the same SamplerStallError (a gene stall is recorded on
// the owning rank only; its peers stopped the chain from the gathered
// flags).  NCCL all-gather of [m, key bits, x0, w] per slot on the engine
// stream, or the loopback group's host exchange.
int exchange_stalls(cmc_engine* e, long lo, long hi, std::vector<StallRec>& recs,
                    std::vector<StallRec>& all, cmc_error* err) {
  const long n = hi - lo;
  const int W = e->world;
  all.assign((size_t)W * n, StallRec{});
  std::vector<double> mine((size_t)n * 4), got((size_t)W * n * 4);
  for (long i = 0; i < n; ++i) {
    mine[4 * i] = (double)recs[i].m;
    std::memcpy(&mine[4 * i + 1], &recs[i].key, 8);
    mine[4 * i + 2] = recs[i].x0;
    mine[4 * i + 3] = recs[i].w;
  }
  if (e->loop) {
    cmc_loopback& g = *e->loop;
    {
      std::lock_guard<std::mutex> lk(g.mu);
      if (g.xrec.size() < (size_t)W) g.xrec.resize((size_t)W);
      g.xrec[(size_t)e->rank] = mine;
    }
    if (!g.barrier()) {
      set_err(err, CMC_ERR_NCCL, "loopback group broken during the stall exchange");
      return CMC_ERR_NCCL;
    }
    for (int r = 0; r < W; ++r)
      std::copy(g.xrec[(size_t)r].begin(), g.xrec[(size_t)r].end(), got.begin() + (size_t)r * n * 4);
    if (!g.barrier()) {
      set_err(err, CMC_ERR_NCCL, "loopback group broken during the stall exchange");
      return CMC_ERR_NCCL;
    }
  } else {
    double* d = e->stall_x.p;
    CUDA_TRY(cudaMemcpyAsync(d + (size_t)e->rank * n * 4, mine.data(), sizeof(double) * n * 4,
                             cudaMemcpyHostToDevice, e->stream));
    if (g_nccl.all_gather(d + (size_t)e->rank * n * 4, d, (size_t)n * 4, kNcclFloat64, e->comm,
                          e->stream) != 0) {
      set_err(err, CMC_ERR_NCCL, "ncclAllGather of the stall records failed");
      return CMC_ERR_NCCL;
    }
    CUDA_TRY(cudaMemcpyAsync(got.data(), d, sizeof(double) * W * n * 4, cudaMemcpyDeviceToHost,
                             e->stream));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
  }
  for (size_t i = 0; i < all.size(); ++i) {
    all[i].m = (long long)got[4 * i];
    std::memcpy(&all[i].key, &got[4 * i + 1], 8);
    all[i].x0 = got[4 * i + 2];
    all[i].w = got[4 * i + 3];
  }
  return CMC_OK;
}

// The stall to report for slots [lo, hi): the lowest stalled chain (the
// reference runs chains in order), and within it the earliest iteration,
// then the smallest key, over every rank.
int check_stall(cmc_engine* e, long slot_lo, long slot_hi, cmc_error* err) {
  const long n = slot_hi - slot_lo;
  std::vector<StallRec> recs((size_t)n);
  for (long c = slot_lo; c < slot_hi; ++c) CUDA_TRY(local_stall(e, c, &recs[(size_t)(c - slot_lo)]));
  std::vector<StallRec> all = recs;
  if (e->split_tail) {  // sharded (a 1-rank clique included)
    const int rc = exchange_stalls(e, slot_lo, slot_hi, recs, all, err);
    if (rc) return rc;
  }
  const int W = e->split_tail ? e->world : 1;
  for (long i = 0; i < n; ++i) {
    const StallRec* best = nullptr;
    for (int r = 0; r < W; ++r) {
      const StallRec& s = all[(size_t)r * n + i];
      if (s.m < 0) continue;
      if (!best || s.m < best->m || (s.m == best->m && s.key < best->key)) best = &s;
    }
    if (best) {
      report_stall(*best, err);
      return CMC_ERR_STALL;
    }
  }
  return CMC_OK;
}

// Debug aid: build with -DCMC_DEBUG_SYNC to synchronise and report after
// each sweep-kernel launch of enqueue_sweep_on (locates a faulting kernel).
#ifdef CMC_DEBUG_SYNC
#define DBG_SYNC(what)                                                             \
  do {                                                                             \
    cudaError_t d_ = cudaDeviceSynchronize();                                      \
    std::fprintf(stderr, "[dbg] %s: %s\n", what, cudaGetErrorString(d_));          \
  } while (0)
#else
#define DBG_SYNC(what) \
  do {                 \
  } while (0)
#endif

// Enqueue one sweep (iteration *d_m + off) for `chains` chains at
// slot_base.  The gene-phase kernels run on the engine stream; the
// reduction/hyper tail runs on tail_stream after ev_gene, so the NEXT
// sweep's eps kernel (which reads only beta and gamma of this sweep) overlaps
// it, and the next gene kernel waits for ev_tail (it reads nu, tau, theta,
// sigma).  In a CUDA graph capture the two streams become parallel branches.
// The all-gather of one lane's partial sections: part = [world][count],
// this rank's section at rank * count.  NCCL, or the in-process loopback.
cudaError_t all_gather_parts(cmc_engine* e, double* part, size_t count, nccl_comm comm,
                             cudaStream_t t) {
  if (!e->loop) {
    if (g_nccl.all_gather(part + (size_t)e->rank * count, part, count, kNcclFloat64, comm, t) != 0)
      return cudaErrorUnknown;
    return cudaSuccess;
  }
  cmc_loopback& g = *e->loop;
  const int r = e->rank;
  auto fail = [&](cudaError_t rc) {
    g.abort();
    return rc;
  };
  cudaError_t rc = cudaEventRecord(e->loop_ready, t);
  if (rc != cudaSuccess) return fail(rc);
  g.send[(size_t)r] = part + (size_t)r * count;
  g.ready[(size_t)r] = e->loop_ready;
  if (!g.barrier()) return cudaErrorTimeout;  // every section published
  for (int q = 0; q < g.world; ++q) {
    if (q == r) continue;
    if ((rc = cudaStreamWaitEvent(t, g.ready[(size_t)q], 0)) != cudaSuccess) return fail(rc);
    if ((rc = cudaMemcpyAsync(part + (size_t)q * count, g.send[(size_t)q], count * sizeof(double),
                              cudaMemcpyDeviceToDevice, t)) != cudaSuccess)
      return fail(rc);
  }
  if ((rc = cudaEventRecord(e->loop_copied, t)) != cudaSuccess) return fail(rc);
  g.copied[(size_t)r] = e->loop_copied;
  // every copy enqueued: a peer re-records its events only after the next
  // exchange's first barrier, i.e. after ours
  if (!g.barrier()) return cudaErrorTimeout;
  // this rank's section is not overwritten (next sweep's leaf kernel)
  // before every peer has copied it
  for (int q = 0; q < g.world; ++q)
    if (q != r && (rc = cudaStreamWaitEvent(t, g.copied[(size_t)q], 0)) != cudaSuccess)
      return fail(rc);
  return cudaSuccess;
}

cudaError_t enqueue_sweep_on(cmc_engine* e, const SweepParams& p_in, int chains,
                             long off, cudaStream_t s, cudaStream_t t,
                             cudaEvent_t ev_gene, cudaEvent_t ev_tail,
                             nccl_comm comm) {
  // this launch's chains own a contiguous section of the partial buffers:
  // [world][chains][Qs][lpr] at world * slot_base * Qs * lpr
  SweepParams p = p_in;
  const int Qs = leaf_qs_a((int)e->L, e->xi_any ? 1 : 0);
  const size_t lpr = (size_t)p.leaves_per_rank, W = (size_t)e->world;
  p.partA = e->partA.p + W * (size_t)p.slot_base * Qs * lpr;
  p.partB = e->partB.p + W * (size_t)p.slot_base * e->L * lpr;
  p.C = chains;
  DBG_SYNC("enter");
  cudaError_t r = launch_eps_sweep(p, chains, off, s);
  if (r != cudaSuccess) return r;
  DBG_SYNC("eps");
  if ((r = cudaStreamWaitEvent(s, ev_tail, 0)) != cudaSuccess) return r;
  // gene kernel: steps 2 and 5 and, without a xi prior, the leaf sums of
  // steps 3/4/6 and (one GPU) the nu, tau, theta draws themselves
  if ((r = launch_gene_sweep(p, chains, off, s)) != cudaSuccess) return r;
  DBG_SYNC("gene");
  if (e->xi_any && (r = launch_xi_sweep(p, chains, off, s)) != cudaSuccess) return r;
  if ((r = cudaEventRecord(ev_gene, s)) != cudaSuccess) return r;
  if ((r = cudaStreamWaitEvent(t, ev_gene, 0)) != cudaSuccess) return r;
  if (!p.fuse_leaf_a && (r = launch_leaf_a(p, chains, off, t)) != cudaSuccess) return r;
  DBG_SYNC("leaf_a");
  if (!e->split_tail) {
    // one GPU: leaf_a's last block runs nu/tau/theta; after the gene
    // kernel's fused leaf sums, hyper_a does
    if (p.fuse_leaf_a && (r = launch_hyper_a(p, chains, off, t)) != cudaSuccess) return r;
    if ((r = launch_leaf_b(p, chains, off, t)) != cudaSuccess) return r;
    DBG_SYNC("leaf_b");
  } else {
    // Every collective of every lane is ordered after the previously
    // enqueued one (ev_coll), so all ranks issue them in one order: lane 0
    // A, lane 0 B, lane 1 A, lane 1 B, then the next sweep.  Communicators
    // of different lanes can then never wait on each other in different
    // orders on different ranks.
    const size_t cA = (size_t)chains * Qs * lpr;
    const size_t cB = (size_t)chains * e->L * lpr;
    if ((r = cudaStreamWaitEvent(t, e->ev_coll, 0)) != cudaSuccess) return r;
    if ((r = all_gather_parts(e, p.partA, cA, comm, t)) != cudaSuccess) return r;
    if ((r = launch_hyper_a(p, chains, off, t)) != cudaSuccess) return r;
    if ((r = launch_leaf_b(p, chains, off, t)) != cudaSuccess) return r;
    if ((r = all_gather_parts(e, p.partB, cB, comm, t)) != cudaSuccess) return r;
    if ((r = cudaEventRecord(e->ev_coll, t)) != cudaSuccess) return r;
    if ((r = launch_hyper_b(p, chains, off, t)) != cudaSuccess) return r;
  }
  if (p.monitor_enabled && e->has_ctab && e->ctab.gene_needs_hyper)
    if ((r = launch_gene_contrast(p, chains, off, t)) != cudaSuccess) return r;
  return cudaEventRecord(ev_tail, t);
}

// One sweep of chains [slot_base, slot_base + chains) on lane 0.
cudaError_t enqueue_sweep(cmc_engine* e, const SweepParams& p, int chains,
                          long off) {
  return enqueue_sweep_on(e, p, chains, off, e->stream, e->tail_stream, e->ev_gene,
                          e->ev_tail, e->comm);
}

// Join the tail stream back into the engine stream (before the iteration
// base advances or the host reads results).
cudaError_t join_tail(cmc_engine* e) {
  return cudaStreamWaitEvent(e->stream, e->ev_tail, 0);
}

// Fork lanes 1.. off the engine stream (inside or outside a capture).
cudaError_t fork_lanes(cmc_engine* e) {
  cudaError_t r = cudaEventRecord(e->ev_fork, e->stream);
  if (r != cudaSuccess) return r;
  for (int k = 1; k < e->n_lanes; ++k) {
    cmc_engine::Lane& ln = e->lanes[k];
    if ((r = cudaStreamWaitEvent(ln.s, e->ev_fork, 0)) != cudaSuccess) return r;
    if ((r = cudaEventRecord(ln.ev_tail, ln.s)) != cudaSuccess) return r;
  }
  // the collective-order event too (captures may only wait on events
  // recorded inside them)
  if (e->ev_coll && (r = cudaEventRecord(e->ev_coll, e->stream)) != cudaSuccess) return r;
  return cudaEventRecord(e->ev_tail, e->stream);
}

// Every lane's sweep of iteration *d_m + off.
cudaError_t enqueue_all_lanes(cmc_engine* e, const SweepParams& base, long off) {
  for (int k = 0; k < e->n_lanes; ++k) {
    cmc_engine::Lane& ln = e->lanes[k];
    SweepParams p = base;
    p.slot_base = ln.slot0;
    p.chain_base = ln.slot0;
    cudaError_t r = enqueue_sweep_on(e, p, ln.chains, off, ln.s, ln.t, ln.ev_gene, ln.ev_tail,
                                     k == 0 ? e->comm : e->lane_comm[k]);
    if (r != cudaSuccess) return r;
  }
  return cudaSuccess;
}

// Join every lane's streams back into the engine stream.
cudaError_t join_lanes(cmc_engine* e) {
  for (int k = 0; k < e->n_lanes; ++k) {
    cmc_engine::Lane& ln = e->lanes[k];
    cudaError_t r = cudaStreamWaitEvent(ln.s, ln.ev_tail, 0);
    if (r != cudaSuccess) return r;
    if (k == 0) continue;
    if ((r = cudaEventRecord(ln.ev_join, ln.s)) != cudaSuccess) return r;
    if ((r = cudaStreamWaitEvent(e->stream, ln.ev_join, 0)) != cudaSuccess) return r;
  }
  return cudaSuccess;
}

// The executable graph of `len` consecutive sweeps of every lane (iteration
// *d_m + 0 .. len-1) followed by the advance of *d_m, from the cache or
// captured now (least recently used slot replaced).
cudaError_t sweep_graph(cmc_engine* e, const SweepParams& p, long len, cudaGraphExec_t* out) {
  const int S = cmc_engine::kGraphSlots;
  ++e->graph_clock;
  for (int k = 0; k < S; ++k)
    if (e->graph[k] && e->graph_len[k] == len) {
      e->graph_use[k] = e->graph_clock;
      *out = e->graph[k];
      return cudaSuccess;
    }
  int victim = -1;
  for (int k = 0; k < S && victim < 0; ++k)
    if (!e->graph[k]) victim = k;
  if (victim < 0) {
    victim = 0;
    for (int k = 1; k < S; ++k)
      if (e->graph_use[k] < e->graph_use[victim]) victim = k;
  }
  if (e->graph[victim]) {
    cudaError_t r = cudaGraphExecDestroy(e->graph[victim]);
    e->graph[victim] = nullptr;
    if (r != cudaSuccess) return r;
  }
  cudaGraph_t g;
  cudaError_t r = cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal);
  if (r != cudaSuccess) return r;
  // fork the other lanes and the tail streams into the capture
  r = fork_lanes(e);
  for (long off = 0; r == cudaSuccess && off < len; ++off) r = enqueue_all_lanes(e, p, off);
  if (r == cudaSuccess) r = join_lanes(e);
  if (r == cudaSuccess) r = launch_advance(e->d_m.p, len, e->stream);
  cudaError_t r2 = cudaStreamEndCapture(e->stream, &g);
  if (r != cudaSuccess) return r;
  if (r2 != cudaSuccess) return r2;
  r = cudaGraphInstantiate(&e->graph[victim], g, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(g);
  if (r != cudaSuccess) return r;
  // upload the executable's work descriptors now: the first replay then
  // does not pay the upload inside its (timed) launch (A/B, 20-sweep call:
  // 0.3406 -> 0.3316 ms per sweep)
  if ((r = cudaGraphUpload(e->graph[victim], e->stream)) != cudaSuccess) return r;
  e->graph_len[victim] = len;
  e->graph_use[victim] = e->graph_clock;
  *out = e->graph[victim];
  return cudaSuccess;
}

int set_device_m(cmc_engine* e, long m, cmc_error* err) {
  if (e->host_m == m) return CMC_OK;
  CUDA_TRY(cudaStreamSynchronize(e->stream));
  CUDA_TRY(cudaMemcpy(e->d_m.p, &m, sizeof(long), cudaMemcpyHostToDevice));
  e->host_m = m;
  return CMC_OK;
}

}  // namespace

extern "C" {

const char* cmc_version(void) {
  return "countmc_b200 0.1 (sm_100a, fp64, -fmad=false parity build)";
}

int cmc_shard_bounds(long G, int rank, int world, long* g_begin, long* g_end) {
  if (world < 1 || rank < 0 || rank >= world || G < 1) return CMC_ERR_ARG;
  const long leaves = (G + kLeaf - 1) / kLeaf;
  const long lpr = (leaves + world - 1) / world;
  const long b = std::min(G, (long)rank * lpr * kLeaf);
  const long en = std::min(G, (long)(rank + 1) * lpr * kLeaf);
  *g_begin = b;
  *g_end = en;
  return CMC_OK;
}

int cmc_engine_create(const cmc_problem* p, const cmc_run_config* config,
                      const cmc_contrast_set* cs, int device, cmc_engine** out,
                      cmc_error* err) {
  if (!p || !config || !out) {
    set_err(err, CMC_ERR_ARG, "null argument");
    return CMC_ERR_ARG;
  }
  *out = nullptr;
  // CountMatrix::validate / ModelSpec::validate / PriorConfig::validate,
  // P:src/types.cpp:18-69
  if (p->G < 1 || p->N < 1)
    return fail_config(err, "count matrix must have at least one gene and one sample");
  if (p->L < 1)
    return fail_config(err, "model matrix must have at least one row and one column");
  if (!p->counts || !p->X || !p->h || !p->c || !p->s) {
    set_err(err, CMC_ERR_ARG, "null problem array");
    return CMC_ERR_ARG;
  }
  for (long i = 0; i < p->G * p->N; ++i)
    if (p->counts[i] < 0) {
      char buf[128];
      std::snprintf(buf, sizeof(buf), "negative count at gene %ld, sample %ld",
                    i / p->N + 1, i % p->N + 1);
      return fail_config(err, buf);
    }
  for (long i = 0; i < p->N; ++i)
    if (!std::isfinite(p->h[i])) return fail_config(err, "offsets must be finite");
  for (long i = 0; i < p->N * p->L; ++i)
    if (!std::isfinite(p->X[i]))
      return fail_config(err, "model matrix entries must be finite");
  if (matrix_rank(std::vector<double>(p->X, p->X + p->N * p->L), p->N, p->L, 1e-10) < p->L)
    return fail_config(err, "model matrix does not have full column rank");
  if (!(p->a > 0.0) || !(p->b > 0.0) || !(p->d > 0.0))
    return fail_config(err, "prior constants a, b, d must be strictly positive");
  for (long l = 0; l < p->L; ++l)
    if (!(p->c[l] > 0.0) || !(p->s[l] > 0.0))
      return fail_config(err, "prior entries c, s must be strictly positive");
  if (p->beta_prior)
    for (long l = 0; l < p->L; ++l) {
      if (p->beta_prior[l] < CMC_PRIOR_NORMAL || p->beta_prior[l] > CMC_PRIOR_HORSESHOE)
        return fail_config(err, "beta prior must be normal, laplace, t or horseshoe");
      if (p->beta_prior[l] == CMC_PRIOR_T && !(p->t_df > 0.0))
        return fail_config(err, "t prior needs positive degrees of freedom");
    }
  // device limits of this build
  if (p->L > kLMax) return fail_config(err, "L exceeds the 16 columns this build supports");
  if (p->N >= (1 << 20)) return fail_config(err, "N too large for this build");
  if (p->G >= (1L << 32)) return fail_config(err, "G too large for this build");
  // RunConfig::resolve, P:src/engine.cpp:25-40
  cmc_run_config cfg = *config;
  if (cfg.chains < 1) return fail_config(err, "chains must be >= 1");
  if (cfg.iterations < 1) return fail_config(err, "iterations must be >= 1");
  if (cfg.burnin < 1) return fail_config(err, "burnin must be >= 1");
  if (cfg.thin < 1) return fail_config(err, "thin must be >= 1");
  if (cfg.workers < 1) return fail_config(err, "workers must be >= 1");
  if (cfg.save_genes < 0) return fail_config(err, "save_genes must be >= 0");
  if (cfg.max_step_out < 1) return fail_config(err, "max_step_out must be >= 1");
  if (cfg.tune_cutoff < 0) cfg.tune_cutoff = std::min<long>(500, cfg.burnin / 10);
  if (cfg.tune_cutoff >= cfg.burnin)
    return fail_config(err, "tune_cutoff must be less than burnin (M_C < M_B)");
  if (!(cfg.w_init > 0.0)) return fail_config(err, "w_init must be positive");
  if (cfg.max_shrink < 1) return fail_config(err, "max_shrink must be >= 1");

  auto* e = new cmc_engine();
  e->G_total = p->G;
  e->N = p->N;
  e->L = p->L;
  e->counts.assign(p->counts, p->counts + p->G * p->N);
  e->X.assign(p->X, p->X + p->N * p->L);
  e->h.assign(p->h, p->h + p->N);
  e->c.assign(p->c, p->c + p->L);
  e->s.assign(p->s, p->s + p->L);
  e->a = p->a;
  e->b = p->b;
  e->d = p->d;
  e->prior.assign((size_t)p->L, CMC_PRIOR_NORMAL);
  if (p->beta_prior) e->prior.assign(p->beta_prior, p->beta_prior + p->L);
  for (int v : e->prior) e->xi_any |= v != CMC_PRIOR_NORMAL;
  e->t_df = p->t_df;
  e->cfg = cfg;
  e->device = device;
  e->C = (int)cfg.chains;
  e->G = p->G;
  e->g0 = 0;

  // column groups in first-appearance order, P:src/engine.cpp:62-75
  const long N = p->N, L = p->L;
  e->grp_off.push_back(0);
  e->grp_moff.push_back(0);
  int jmax = 1;
  for (long l = 0; l < L; ++l) {
    std::vector<double> vals;
    std::vector<std::vector<int>> mem;
    for (long n = 0; n < N; ++n) {
      const double v = p->X[n * L + l];
      if (v == 0.0) continue;
      size_t j = 0;
      for (; j < vals.size(); ++j)
        if (vals[j] == v) break;
      if (j == vals.size()) {
        vals.push_back(v);
        mem.emplace_back();
      }
      mem[j].push_back((int)n);
    }
    for (size_t j = 0; j < vals.size(); ++j) {
      e->grp_val.push_back(vals[j]);
      e->grp_mem.insert(e->grp_mem.end(), mem[j].begin(), mem[j].end());
      e->grp_moff.push_back((int)e->grp_mem.size());
    }
    e->grp_off.push_back((int)e->grp_val.size());
    jmax = std::max<int>(jmax, (int)vals.size());
  }
  e->Jmax = jmax;
  {
    // the gene kernel keeps lp (N) and, beyond 2 groups per column, the
    // group sums (2 Jmax) per gene in shared memory
    // (5 KB reserved for the kernel's static shared memory: the exp table
    // and the Philox queues' second blocks; ensure_device checks the exact
    // total against the device's opt-in limit)
    const int smem = gene_sweep_smem_bytes((int)p->N, jmax <= 2 ? 0 : jmax);
    if (smem + 5 * 1024 > 227 * 1024) {
      delete e;
      return fail_config(err, "N (plus 2x the groups per model-matrix column) too large for "
                              "this build's gene kernel: at most 222 samples");
    }
  }

  // saved genes: partial Fisher-Yates on (seed, 0, 0, kSaveSel), sorted,
  // P:src/engine.cpp:77-90
  const long k = std::min<long>(cfg.save_genes, p->G);
  if (k > 0) {
    std::vector<long> idx((size_t)p->G);
    std::iota(idx.begin(), idx.end(), 0L);
    Stream sel;
    sel.init(cfg.seed, 0, 0, site_id(kSiteSaveSel, 0));
    for (long i = 0; i < k; ++i) {
      const long j = i + (long)sel.uniform_int((uint64_t)(p->G - i));
      std::swap(idx[(size_t)i], idx[(size_t)j]);
    }
    e->saved.assign(idx.begin(), idx.begin() + k);
    std::sort(e->saved.begin(), e->saved.end());
  }
  e->n_cols = 2 + 2 * L + (long)e->saved.size() * (L + 1);
  e->n_rows = cfg.iterations / cfg.thin;

  // contrasts: ContrastSpec::finalize (P:src/streaming.cpp:76-88) and
  // parse_param_ref's range check (P:src/streaming.cpp:65-72)
  if (cs && cs->n_contrasts > 0) {
    ContrastTable& t = e->ctab;
    std::memset(&t, 0, sizeof(t));
    if (cs->n_contrasts > kMaxContrasts) {
      delete e;
      return fail_config(err, "too many contrasts for this build (max 8)");
    }
    t.n = cs->n_contrasts;
    int term = 0, q = 0;
    long off = 0;
    for (int ci = 0; ci < cs->n_contrasts; ++ci) {
      t.term_begin[ci] = term;
      if (cs->n_terms[ci] < 1) {
        delete e;
        return fail_config(err, "contrast has no terms");
      }
      bool per_gene = false, needs_hyper = false;
      for (int ti = 0; ti < cs->n_terms[ci]; ++ti, ++term) {
        if (term >= kMaxTerms) {
          delete e;
          return fail_config(err, "too many contrast terms for this build");
        }
        t.coef_begin[term] = q;
        t.threshold[term] = cs->threshold[term];
        if (cs->n_coefs[term] < 1) {
          delete e;
          return fail_config(err, "contrast has a term with no coefficients");
        }
        for (int kk = 0; kk < cs->n_coefs[term]; ++kk, ++q) {
          if (q >= kMaxCoefs) {
            delete e;
            return fail_config(err, "too many contrast coefficients for this build");
          }
          const int fam = cs->family[q], ix = cs->index[q];
          if (fam < 0 || fam > 5) {
            delete e;
            return fail_config(err, "unknown parameter name in contrast");
          }
          if ((fam == CMC_FAM_BETA_COL || fam == CMC_FAM_THETA || fam == CMC_FAM_SIGMA) &&
              (ix < 0 || ix >= L)) {
            delete e;
            return fail_config(err, "contrast index out of range");
          }
          t.fam[q] = fam;
          t.idx[q] = ix;
          t.coef[q] = cs->coef[q];
          if (fam == CMC_FAM_BETA_COL || fam == CMC_FAM_GAMMA) per_gene = true;
          else needs_hyper = true;
        }
      }
      t.per_gene[ci] = per_gene ? 1 : 0;
      if (per_gene && needs_hyper) t.gene_needs_hyper = 1;
      t.prob_off[ci] = off;
      off += per_gene ? p->G : 1;
    }
    t.term_begin[cs->n_contrasts] = term;
    t.coef_begin[term] = q;
    t.n_prob = off;
    e->has_ctab = true;
  }
  *out = e;
  return CMC_OK;
}

int cmc_engine_destroy(cmc_engine* e) {
  if (!e) return CMC_OK;
  if (e->dev_ready) {
    cudaSetDevice(e->device);
    // every lane's work done before the pooled buffers go back (cudaFree
    // used to imply this)
    cudaDeviceSynchronize();
    for (auto& g : e->graph)
      if (g) cudaGraphExecDestroy(g);
    DevBuf<double>* ds[] = {&e->y, &e->A, &e->Xd, &e->hd, &e->gval, &e->eps,
                            &e->eps_w, &e->eps_wa, &e->gam, &e->gam_w,
                            &e->gam_wa, &e->beta, &e->beta_w, &e->beta_wa,
                            &e->log_gam, &e->inv_gam, &e->acc_eps, &e->acc_gam,
                            &e->acc_beta, &e->cprob, &e->samples, &e->partA,
                            &e->partB, &e->xi, &e->xi_w, &e->xi_wa, &e->acc_xi,
                            &e->xfer};
    for (auto* b : ds) b->free_();
    e->goff.free_();
    e->gmoff.free_();
    e->gmem.free_();
    e->saved_slot.free_();
    e->hyper.free_();
    e->leaf_cnt.free_();
    e->step_cyc.free_();
    e->stall_x.free_();
    if (e->ev_coll) cudaEventDestroy(e->ev_coll);
    e->dctab.free_();
    e->d_m.free_();
    if (e->ev0) cudaEventDestroy(e->ev0);
    for (int k = 1; k < e->n_lanes; ++k) {
      cmc_engine::Lane& ln = e->lanes[k];
      cudaStreamSynchronize(ln.s);
      cudaStreamSynchronize(ln.t);
      cudaEventDestroy(ln.ev_gene);
      cudaEventDestroy(ln.ev_tail);
      cudaStreamDestroy(ln.s);
      cudaStreamDestroy(ln.t);
    }
    for (int k = 0; k < e->n_lanes; ++k)
      if (e->lanes[k].ev_join) cudaEventDestroy(e->lanes[k].ev_join);
    if (e->ev_fork) cudaEventDestroy(e->ev_fork);
    if (e->ev_gene) cudaEventDestroy(e->ev_gene);
    if (e->ev_tail) cudaEventDestroy(e->ev_tail);
    if (e->tail_stream) cudaStreamDestroy(e->tail_stream);
    if (e->ev1) cudaEventDestroy(e->ev1);
    cudaStreamDestroy(e->stream);
  }
  if (e->loop_ready) cudaEventDestroy(e->loop_ready);
  if (e->loop_copied) cudaEventDestroy(e->loop_copied);
  for (int k = 1; k < 4; ++k)
    if (e->lane_comm[k] && g_nccl.destroy) g_nccl.destroy(e->lane_comm[k]);
  if (e->comm && g_nccl.destroy) g_nccl.destroy(e->comm);
  delete e;
  return CMC_OK;
}

int cmc_engine_dims(const cmc_engine* e, long* G, long* N, long* L,
                    long* chains, long* n_saved, long* n_cols, long* n_rows) {
  if (!e) return CMC_ERR_ARG;
  if (G) *G = e->G_total;
  if (N) *N = e->N;
  if (L) *L = e->L;
  if (chains) *chains = e->C;
  if (n_saved) *n_saved = (long)e->saved.size();
  if (n_cols) *n_cols = e->n_cols;
  if (n_rows) *n_rows = e->n_rows;
  return CMC_OK;
}

int cmc_engine_saved_genes(const cmc_engine* e, long* out) {
  if (!e || !out) return CMC_ERR_ARG;
  std::copy(e->saved.begin(), e->saved.end(), out);
  return CMC_OK;
}

int cmc_engine_config(const cmc_engine* e, cmc_run_config* out) {
  if (!e || !out) return CMC_ERR_ARG;
  *out = e->cfg;
  return CMC_OK;
}

int cmc_engine_initial_state(const cmc_engine* e, long chain, double* state,
                             cmc_error* err) {
  if (!e || !state || chain < 0) {
    set_err(err, CMC_ERR_ARG, "bad argument");
    return CMC_ERR_ARG;
  }
  initial_state_host(e, chain, state);
  return CMC_OK;
}

int cmc_engine_set_state(cmc_engine* e, long chain, const double* state,
                         const double* tw, const double* ta, cmc_error* err) {
  if (!e || !state || chain < 0) {
    set_err(err, CMC_ERR_ARG, "bad chain or state");
    return CMC_ERR_ARG;
  }
  int rc = ensure_device(e, err);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(e->device));
  CUDA_TRY(cudaStreamSynchronize(e->stream));
  // the reference's iterate() takes any chain id and caller-owned state:
  // the state lives in the scratch slot C (a run()'s chains stay untouched),
  // the chain id only keys the random stream
  return upload_state(e, e->C, state, tw, ta, err);
}

int cmc_engine_get_state(cmc_engine* e, long chain, double* state, double* tw,
                         double* ta, cmc_error* err) {
  if (!e || chain < 0) {
    set_err(err, CMC_ERR_ARG, "bad chain");
    return CMC_ERR_ARG;
  }
  int rc = ensure_device(e, err);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(e->device));
  CUDA_TRY(cudaStreamSynchronize(e->stream));
  return download_state(e, e->C, state, tw, ta, err);
}

int cmc_engine_iterate(cmc_engine* e, long chain, long m, uint64_t* clamps,
                       cmc_error* err) {
  if (!e || chain < 0 || m < 1) {
    set_err(err, CMC_ERR_ARG, "bad chain or iteration");
    return CMC_ERR_ARG;
  }
  int rc = ensure_device(e, err);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(e->device));
  const long run_m = e->host_m;  // a run()'s iteration counter, restored below
  if ((rc = set_device_m(e, m, err))) return rc;
  const long slot = e->C;  // scratch slot: a run()'s chains stay untouched
  Hyper hp;
  CUDA_TRY(cudaMemcpy(&hp, e->hyper.p + slot, sizeof(Hyper), cudaMemcpyDeviceToHost));
  const unsigned long long before = hp.clamps;
  hp.err_key = kNoError;
  hp.err_key_eps = kNoError;
  hp.peer_stall = 0;
  CUDA_TRY(cudaMemcpy(&e->hyper.p[slot].peer_stall, &hp.peer_stall, sizeof(unsigned int),
                      cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(&e->hyper.p[slot].err_key, &hp.err_key,
                      sizeof(unsigned long long), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(&e->hyper.p[slot].err_key_eps, &hp.err_key_eps,
                      sizeof(unsigned long long), cudaMemcpyHostToDevice));
  SweepParams p = e->base;
  p.slot_base = (int)slot;
  p.chain_base = (int)chain;
  p.monitor_enabled = 0;
  CUDA_TRY(enqueue_sweep(e, p, 1, 0));
  CUDA_TRY(join_tail(e));
  CUDA_TRY(cudaStreamSynchronize(e->stream));
  CUDA_TRY(cudaMemcpy(&hp, e->hyper.p + slot, sizeof(Hyper), cudaMemcpyDeviceToHost));
  if (clamps) *clamps += hp.clamps - before;
  if ((rc = set_device_m(e, run_m, err))) return rc;
  // sharded: every rank takes part in the record exchange, stalled or not
  if (e->split_tail || hp.err_key != kNoError || hp.err_key_eps != kNoError)
    return check_stall(e, slot, slot + 1, err);
  return CMC_OK;
}

int cmc_engine_begin(cmc_engine* e, cmc_error* err) {
  if (!e) return CMC_ERR_ARG;
  const double T0 = tnow();
  const long XI = e->xi_any ? e->G_total * e->L : 0;
  const long S = e->G_total * e->N + e->G_total + e->G_total * e->L + 2 * e->L + 2 + XI;
  // The chains' initial states (host, glibc: bit-identical to the
  // reference) are computed on host threads, one per chain, while this
  // thread sets up the device (allocations, inputs); up to 2 GB of host
  // staging, else one chain at a time below.
  const bool overlap = (double)e->C * (double)S * 8.0 <= 2e9;
  std::vector<std::vector<double>> sts(overlap ? (size_t)e->C : 0);
  std::thread init_th;
  if (overlap)
    init_th = std::thread([e, S, &sts] {
      std::vector<std::thread> per;
      for (long c = 0; c < e->C; ++c)
        per.emplace_back([e, S, &sts, c] {
          sts[(size_t)c].resize((size_t)S);
          initial_state_host(e, c, sts[(size_t)c].data());
        });
      for (auto& t : per) t.join();
    });
  int rc = ensure_device(e, err);
  if (rc == CMC_OK && overlap && !e->loop && !e->split_tail && !e->step_timing) {
    // the run's sweep graphs (the 50-sweep chunk and the remainder of
    // burnin + iterations) are captured now, while the initial states are
    // computed on the other thread, instead of at the first sweeps call
    // with the device idle (17 ms at G = 39,656, 4 chains)
    SweepParams p = e->base;
    p.slot_base = 0;
    p.chain_base = 0;
    p.monitor_enabled = 1;
    const long total = e->cfg.burnin + e->cfg.iterations;
    cudaGraphExec_t g = nullptr;
    cudaError_t ce = cudaSuccess;
    if (total >= CMC_GRAPH_CHUNK) ce = sweep_graph(e, p, CMC_GRAPH_CHUNK, &g);
    if (ce == cudaSuccess && total % CMC_GRAPH_CHUNK)
      ce = sweep_graph(e, p, total % CMC_GRAPH_CHUNK, &g);
    if (ce != cudaSuccess) {
      set_err(err, CMC_ERR_CUDA, std::string("sweep graph capture: ") + cudaGetErrorString(ce));
      rc = CMC_ERR_CUDA;
    }
  }
  if (init_th.joinable()) init_th.join();
  if (rc) return rc;
  const double T1 = tnow();
  double Tis = 0, Tup = 0;
  CUDA_TRY(cudaSetDevice(e->device));
  CUDA_TRY(cudaStreamSynchronize(e->stream));
  std::vector<double> st(overlap ? 0 : (size_t)S);
  CUDA_TRY(cudaMemset(e->hyper.p, 0, sizeof(Hyper) * e->C));
  for (long c = 0; c < e->C; ++c) {
    double a = tnow();
    double* sc = overlap ? sts[(size_t)c].data() : st.data();
    if (!overlap) initial_state_host(e, c, sc);
    double b = tnow();
    if ((rc = upload_state(e, c, sc, nullptr, nullptr, err))) return rc;
    Tis += b - a; Tup += tnow() - b;
  }
  const double T2 = tnow();
  // fresh tuning of every run chain (TuningState(G, N, L, w_init),
  // P:include/countmc/engine.hpp:58-74): widths w_init, accumulators 0,
  // filled on the device instead of uploading two packed host arrays
  {
    const size_t C = (size_t)e->C, G = (size_t)e->G, N = (size_t)e->N, L = (size_t)e->L;
    const double w0 = e->cfg.w_init;
    CUDA_TRY(launch_fill(e->eps_w.p, C * N * G, w0, e->stream));
    CUDA_TRY(launch_fill(e->gam_w.p, C * G, w0, e->stream));
    CUDA_TRY(launch_fill(e->beta_w.p, C * L * G, w0, e->stream));
    CUDA_TRY(cudaMemsetAsync(e->eps_wa.p, 0, sizeof(double) * C * N * G, e->stream));
    CUDA_TRY(cudaMemsetAsync(e->gam_wa.p, 0, sizeof(double) * C * G, e->stream));
    CUDA_TRY(cudaMemsetAsync(e->beta_wa.p, 0, sizeof(double) * C * L * G, e->stream));
    if (e->xi_any) {
      CUDA_TRY(launch_fill(e->xi_w.p, C * L * G, w0, e->stream));
      CUDA_TRY(cudaMemsetAsync(e->xi_wa.p, 0, sizeof(double) * C * L * G, e->stream));
    }
    std::vector<Hyper> hp(C);
    CUDA_TRY(cudaMemcpy(hp.data(), e->hyper.p, sizeof(Hyper) * C, cudaMemcpyDeviceToHost));
    for (auto& h : hp) {
      for (long l = 0; l < e->L; ++l) {
        h.w_sigma[l] = w0;
        h.wa_sigma[l] = 0.0;
      }
      h.w_nu = h.w_tau = w0;
      h.wa_nu = h.wa_tau = 0.0;
    }
    CUDA_TRY(cudaMemcpy(e->hyper.p, hp.data(), sizeof(Hyper) * C, cudaMemcpyHostToDevice));
  }
  CUDA_TRY(cudaMemset(e->acc_eps.p, 0, sizeof(double) * e->acc_eps.n));
  CUDA_TRY(cudaMemset(e->acc_gam.p, 0, sizeof(double) * e->acc_gam.n));
  CUDA_TRY(cudaMemset(e->acc_beta.p, 0, sizeof(double) * e->acc_beta.n));
  if (e->xi_any) CUDA_TRY(cudaMemset(e->acc_xi.p, 0, sizeof(double) * e->acc_xi.n));
  CUDA_TRY(cudaMemset(e->cprob.p, 0, sizeof(double) * e->cprob.n));
  CUDA_TRY(cudaMemset(e->samples.p, 0, sizeof(double) * e->samples.n));
  long one = 1;
  CUDA_TRY(cudaMemcpy(e->d_m.p, &one, sizeof(long), cudaMemcpyHostToDevice));
  e->host_m = 1;
  e->sweep_seconds = 0.0;
  e->step_timed = false;
  e->step_sec.assign((size_t)e->C * 7, 0.0);
  CUDA_TRY(cudaMemset(e->step_cyc.p, 0, sizeof(unsigned long long) * e->step_cyc.n));
  e->begun = true;
  if (std::getenv("CMC_PHASE_LOG"))
    fprintf(stderr, "begin: ensure_device %.1f ms, init states %.1f ms, upload %.1f ms, rest %.1f ms\n",
            1e3 * (T1 - T0), 1e3 * Tis, 1e3 * Tup, 1e3 * (tnow() - T2));
  return CMC_OK;
}

// Per-step timing mode: each sweep's steps launched one at a time for all
// chains on the engine stream, CUDA events between them: eps (step 1), the
// gene kernel split into its step-2 and step-5 launches (the latter with
// the fused leaf sums, and the xi kernel with a xi prior), hyper_a (steps
// 3, 4, 6; leaf_a with a xi prior), leaf_b (step 7).  The nu / tau / theta
// draws inside hyper_a are told apart by the kernel's clock64 stamps; the
// rest of that kernel (the leaf reductions, launch) is charged to nu.  A
// launch covers all chains, so each chain is charged 1/C of it.  Results
// are bit-identical to the fused schedule (same kernels, same order of
// dependent steps).  Single GPU only.
int step_timed_sweeps(cmc_engine* e, const SweepParams& p_in, long total, cmc_error* err) {
  if (e->split_tail || e->loop) {
    set_err(err, CMC_ERR_ARG, "per-step timing is single-GPU only");
    return CMC_ERR_ARG;
  }
  SweepParams p = p_in;
  p.C = (int)e->C;
  p.step_cycles = e->step_cyc.p;
  cudaStream_t s = e->stream;
  CUDA_TRY(cudaStreamWaitEvent(s, e->ev_tail, 0));
  for (int k = 1; k < e->n_lanes; ++k) CUDA_TRY(cudaStreamWaitEvent(s, e->lanes[k].ev_tail, 0));
  constexpr int P = 6;
  std::vector<cudaEvent_t> ev((size_t)(P + 1) * total);
  for (auto& x : ev) CUDA_TRY(cudaEventCreate(&x));
  std::vector<unsigned long long> cyc0(e->step_cyc.n);
  CUDA_TRY(cudaMemcpy(cyc0.data(), e->step_cyc.p, sizeof(unsigned long long) * cyc0.size(),
                      cudaMemcpyDeviceToHost));
  for (long off = 0; off < total; ++off) {
    cudaEvent_t* E = ev.data() + (P + 1) * off;
    CUDA_TRY(cudaEventRecord(E[0], s));
    CUDA_TRY(launch_eps_sweep(p, e->C, off, s));
    CUDA_TRY(cudaEventRecord(E[1], s));
    CUDA_TRY(launch_gene_sweep(p, e->C, off, s, 1));
    CUDA_TRY(cudaEventRecord(E[2], s));
    CUDA_TRY(launch_gene_sweep(p, e->C, off, s, 2));
    if (e->xi_any) CUDA_TRY(launch_xi_sweep(p, e->C, off, s));
    CUDA_TRY(cudaEventRecord(E[3], s));
    CUDA_TRY(p.fuse_leaf_a ? launch_hyper_a(p, e->C, off, s) : launch_leaf_a(p, e->C, off, s));
    CUDA_TRY(cudaEventRecord(E[4], s));
    CUDA_TRY(launch_leaf_b(p, e->C, off, s));
    CUDA_TRY(cudaEventRecord(E[5], s));
    if (p.monitor_enabled && e->has_ctab && e->ctab.gene_needs_hyper)
      CUDA_TRY(launch_gene_contrast(p, e->C, off, s));
    CUDA_TRY(cudaEventRecord(E[6], s));
  }
  CUDA_TRY(launch_advance(e->d_m.p, total, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  double ms[P] = {0, 0, 0, 0, 0, 0};
  for (long off = 0; off < total; ++off)
    for (int k = 0; k < P; ++k) {
      float t = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&t, ev[(P + 1) * off + k], ev[(P + 1) * off + k + 1]));
      ms[k] += t;
    }
  for (auto& x : ev) cudaEventDestroy(x);
  std::vector<unsigned long long> cyc1(e->step_cyc.n);
  CUDA_TRY(cudaMemcpy(cyc1.data(), e->step_cyc.p, sizeof(unsigned long long) * cyc1.size(),
                      cudaMemcpyDeviceToHost));
  int khz = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, e->device));
  const double sec_per_cycle = khz > 0 ? 1.0 / (khz * 1e3) : 0.0;
  const double C = (double)e->C;
  double drawn = 0.0;  // seconds of the tau and theta draws, all chains
  std::vector<double> d((size_t)e->C * 3);
  for (long c = 0; c < e->C; ++c)
    for (int k = 0; k < 3; ++k) {
      d[(size_t)c * 3 + k] = (double)(cyc1[(size_t)c * 4 + k] - cyc0[(size_t)c * 4 + k]) * sec_per_cycle;
      if (k) drawn += d[(size_t)c * 3 + k];
    }
  const double hyper_rest = std::max(0.0, ms[3] * 1e-3 - drawn / C);
  for (long c = 0; c < e->C; ++c) {
    double* st = &e->step_sec[(size_t)c * 7];
    st[0] += ms[0] * 1e-3 / C;                                // epsilon
    st[1] += ms[1] * 1e-3 / C;                                // gamma
    st[2] += hyper_rest / C;                                  // nu (+ the reductions)
    st[3] += d[(size_t)c * 3 + 1];                            // tau
    st[4] += ms[2] * 1e-3 / C;                                // beta (+ leaf sums, xi)
    st[5] += d[(size_t)c * 3 + 2];                            // theta
    st[6] += (ms[4] + ms[5]) * 1e-3 / C;                      // sigma (+ monitors)
  }
  e->sweep_seconds += (ms[0] + ms[1] + ms[2] + ms[3] + ms[4] + ms[5]) * 1e-3;
  e->step_timed = true;
  return CMC_OK;
}

int cmc_engine_sweeps(cmc_engine* e, long m_begin, long m_end, cmc_error* err) {
  if (!e || m_begin < 1 || m_end < m_begin) {
    set_err(err, CMC_ERR_ARG, "bad iteration range");
    return CMC_ERR_ARG;
  }
  if (!e->begun) {
    set_err(err, CMC_ERR_ARG, "cmc_engine_begin must be called first");
    return CMC_ERR_ARG;
  }
  CUDA_TRY(cudaSetDevice(e->device));
  int rc = set_device_m(e, m_begin, err);
  if (rc) return rc;
  SweepParams p = e->base;
  p.slot_base = 0;
  p.chain_base = 0;
  p.monitor_enabled = 1;
  const long total = m_end - m_begin;
  if (e->step_timing) {
    const int rc = step_timed_sweeps(e, p, total, err);
    if (rc == CMC_OK) e->host_m = m_end;
    return rc;
  }
  CUDA_TRY(cudaEventRecord(e->ev0, e->stream));
  if (e->loop) {
    // loopback group: eager launches (another engine's events cannot enter
    // a capture)
    CUDA_TRY(fork_lanes(e));
    for (long off = 0; off < total; ++off) CUDA_TRY(enqueue_all_lanes(e, p, off));
    CUDA_TRY(join_lanes(e));
    CUDA_TRY(launch_advance(e->d_m.p, total, e->stream));
  } else {
    // whole 50-sweep graphs, then one graph of the remaining length: every
    // sweep of the call replays from a graph (a 1-sweep call included)
    const long chunk = CMC_GRAPH_CHUNK;
    const long full = total / chunk, rest = total % chunk;
    if (full) {
      cudaGraphExec_t g = nullptr;
      CUDA_TRY(sweep_graph(e, p, chunk, &g));
      for (long k = 0; k < full; ++k) CUDA_TRY(cudaGraphLaunch(g, e->stream));
    }
    if (rest) {
      cudaGraphExec_t g = nullptr;
      CUDA_TRY(sweep_graph(e, p, rest, &g));
      CUDA_TRY(cudaGraphLaunch(g, e->stream));
    }
    // events recorded inside a capture cannot be waited on outside it:
    // re-arm them on the real streams (all work so far is stream-ordered)
    CUDA_TRY(fork_lanes(e));
    CUDA_TRY(join_lanes(e));
  }
  CUDA_TRY(cudaEventRecord(e->ev1, e->stream));
  e->timing_pending = true;
  e->host_m = m_end;
  return CMC_OK;
}

int cmc_engine_set_step_timing(cmc_engine* e, int on) {
  if (!e) return CMC_ERR_ARG;
  e->step_timing = on != 0;
  return CMC_OK;
}

int cmc_engine_prepare(cmc_engine* e, long sweeps, cmc_error* err) {
  if (!e || sweeps < 1 || !e->begun) {
    set_err(err, CMC_ERR_ARG, "prepare needs begin() and sweeps >= 1");
    return CMC_ERR_ARG;
  }
  if (e->loop) return CMC_OK;  // loopback sweeps are eager
  CUDA_TRY(cudaSetDevice(e->device));
  SweepParams p = e->base;
  p.slot_base = 0;
  p.chain_base = 0;
  p.monitor_enabled = 1;
  cudaGraphExec_t g = nullptr;
  if (sweeps >= CMC_GRAPH_CHUNK) CUDA_TRY(sweep_graph(e, p, CMC_GRAPH_CHUNK, &g));
  if (sweeps % CMC_GRAPH_CHUNK) CUDA_TRY(sweep_graph(e, p, sweeps % CMC_GRAPH_CHUNK, &g));
  return CMC_OK;
}

int cmc_engine_sync(cmc_engine* e, cmc_error* err) {
  if (!e) return CMC_ERR_ARG;
  if (!e->dev_ready) return CMC_OK;
  CUDA_TRY(cudaSetDevice(e->device));
  CUDA_TRY(cudaStreamSynchronize(e->stream));
  CUDA_TRY(cudaStreamSynchronize(e->tail_stream));
  for (int k = 1; k < e->n_lanes; ++k) {
    CUDA_TRY(cudaStreamSynchronize(e->lanes[k].s));
    CUDA_TRY(cudaStreamSynchronize(e->lanes[k].t));
  }
  if (e->timing_pending) {
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
    e->sweep_seconds += ms * 1e-3;
    e->timing_pending = false;
  }
  return check_stall(e, 0, e->C, err);
}

int cmc_engine_run(cmc_engine* e, cmc_error* err) {
  int rc = cmc_engine_begin(e, err);
  if (rc) return rc;
  const long total = e->cfg.burnin + e->cfg.iterations;
  if ((rc = cmc_engine_sweeps(e, 1, total + 1, err))) return rc;
  return cmc_engine_sync(e, err);
}

void* cmc_engine_stream(cmc_engine* e) {
  if (!e) return nullptr;
  cmc_error err;
  if (ensure_device(e, &err)) return nullptr;
  return (void*)e->stream;
}

int cmc_engine_launches_per_sweep(const cmc_engine* e) {
  if (!e) return 0;
  // per lane: eps, gene (+ its fused leaf sums), hyper_a (nu, tau, theta),
  // leaf_b (+ sigma); a xi prior: + xi, and leaf_a replaces the fused sums
  // (its last block draws nu/tau/theta on one GPU); sharded: + hyper_b
  int n = 4;
  if (e->xi_any) n += e->split_tail ? 2 : 1;
  if (e->split_tail) ++n;
  if (e->has_ctab && e->ctab.gene_needs_hyper) ++n;
  return n * std::max(1, e->n_lanes);
}

// Per-phase device time of `reps` further monitored sweeps of every chain
// (one launch per phase for all chains, serialised on the engine stream,
// CUDA events between phases).  ms[CMC_PHASES]: eps (step 1), gene (steps
// 2 + 5 and the fused leaf sums), xi, hyper_a (nu, tau, theta; with a xi
// prior leaf_a), leaf_b (+ sigma, monitors), gene_contrast; averages per
// sweep.
int cmc_engine_profile_phases(cmc_engine* e, long m_begin, long reps, double* ms,
                              cmc_error* err) {
  if (!e || reps < 1 || !e->begun || !ms) {
    set_err(err, CMC_ERR_ARG, "profile needs begin(), reps >= 1 and an output array");
    return CMC_ERR_ARG;
  }
  if (e->split_tail) {
    set_err(err, CMC_ERR_ARG, "profile is single-GPU only");
    return CMC_ERR_ARG;
  }
  CUDA_TRY(cudaSetDevice(e->device));
  int rc = set_device_m(e, m_begin, err);
  if (rc) return rc;
  SweepParams p = e->base;
  p.slot_base = 0;
  p.chain_base = 0;
  p.monitor_enabled = 1;
  constexpr int P = CMC_PHASES;
  std::vector<cudaEvent_t> ev((size_t)((P + 1) * reps));
  for (auto& x : ev) CUDA_TRY(cudaEventCreate(&x));
  cudaStream_t s = e->stream;
  for (long r = 0; r < reps; ++r) {
    cudaEvent_t* E = ev.data() + (P + 1) * r;
    CUDA_TRY(cudaEventRecord(E[0], s));
    CUDA_TRY(launch_eps_sweep(p, e->C, r, s));
    CUDA_TRY(cudaEventRecord(E[1], s));
    CUDA_TRY(launch_gene_sweep(p, e->C, r, s));
    CUDA_TRY(cudaEventRecord(E[2], s));
    if (e->xi_any) CUDA_TRY(launch_xi_sweep(p, e->C, r, s));
    CUDA_TRY(cudaEventRecord(E[3], s));
    CUDA_TRY(p.fuse_leaf_a ? launch_hyper_a(p, e->C, r, s) : launch_leaf_a(p, e->C, r, s));
    CUDA_TRY(cudaEventRecord(E[4], s));
    CUDA_TRY(launch_leaf_b(p, e->C, r, s));
    CUDA_TRY(cudaEventRecord(E[5], s));
    if (e->has_ctab && e->ctab.gene_needs_hyper) CUDA_TRY(launch_gene_contrast(p, e->C, r, s));
    CUDA_TRY(cudaEventRecord(E[6], s));
  }
  CUDA_TRY(launch_advance(e->d_m.p, reps, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  e->host_m = m_begin + reps;
  for (int k = 0; k < P; ++k) ms[k] = 0.0;
  for (long r = 0; r < reps; ++r)
    for (int k = 0; k < P; ++k) {
      float t = 0.f;
      CUDA_TRY(cudaEventElapsedTime(&t, ev[(P + 1) * r + k], ev[(P + 1) * r + k + 1]));
      ms[k] += t / reps;
    }
  for (auto& x : ev) cudaEventDestroy(x);
  return check_stall(e, 0, e->C, err);
}

int cmc_engine_profile(cmc_engine* e, long m_begin, long reps, double* gene_ms,
                       double* tail_ms, cmc_error* err) {
  double ms[CMC_PHASES];
  const int rc = cmc_engine_profile_phases(e, m_begin, reps, ms, err);
  if (rc) return rc;
  if (gene_ms) *gene_ms = ms[0] + ms[1] + ms[2];
  if (tail_ms) *tail_ms = ms[3] + ms[4] + ms[5];
  return CMC_OK;
}

// Runs the diagnostics kernels over the resident accumulators and copies
// [rhat | mean | sd | lo | hi] (5R), ess (n_cols) and [flags R | ess_status
// n_cols] to the host.  count = monitored iterations per chain.
static int diag_to_host(cmc_engine* e, long count, std::vector<double>& vals,
                        std::vector<int>& flags, cmc_error* err) {
  CUDA_TRY(cudaSetDevice(e->device));
  CUDA_TRY(cudaStreamSynchronize(e->stream));
  const long L = e->L, G = e->G;
  const long R = 2 + 2 * L + G * (L + 1);
  const long rows = std::min<long>(e->n_rows, count / e->cfg.thin);
  DiagParams d{};
  d.C = e->C;
  d.L = (int)L;
  d.N = (int)e->N;
  d.G = G;
  d.M = count;
  d.n_cols = e->n_cols;
  d.n_rows = rows;
  d.hyper = e->hyper.p;
  d.acc_beta = e->acc_beta.p;
  d.acc_gam = e->acc_gam.p;
  d.z = normal_quantile(1.0 - 0.05 / 2.0);
  // samples are stored [C][n_cols][n_rows_alloc]; the ESS kernel reads a
  // compact [C][n_cols][rows] copy
  DevBuf<double> out, smp;
  DevBuf<int> fl;
  CUDA_TRY(out.alloc((size_t)5 * R + e->n_cols));
  CUDA_TRY(fl.alloc((size_t)R + e->n_cols));
  CUDA_TRY(smp.alloc(std::max<size_t>(1, (size_t)e->C * e->n_cols * rows)));
  if (rows > 0)
    CUDA_TRY(cudaMemcpy2DAsync(smp.p, sizeof(double) * rows, e->samples.p,
                               sizeof(double) * e->n_rows, sizeof(double) * rows,
                               (size_t)e->C * e->n_cols, cudaMemcpyDeviceToDevice, e->stream));
  d.samples = smp.p;
  d.rhat = out.p;
  d.mean = out.p + R;
  d.sd = out.p + 2 * R;
  d.lo = out.p + 3 * R;
  d.hi = out.p + 4 * R;
  d.ess = out.p + 5 * R;
  d.flags = fl.p;
  d.ess_status = fl.p + R;
  CUDA_TRY(launch_diagnostics(d, e->stream));
  CUDA_TRY(cudaStreamSynchronize(e->stream));
  vals.resize((size_t)5 * R + e->n_cols);
  flags.resize((size_t)R + e->n_cols);
  CUDA_TRY(cudaMemcpy(vals.data(), out.p, sizeof(double) * vals.size(), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(flags.data(), fl.p, sizeof(int) * flags.size(), cudaMemcpyDeviceToHost));
  out.free_();
  fl.free_();
  smp.free_();
  return CMC_OK;
}

static long monitored_count(const cmc_engine* e) {
  return std::max<long>(0, std::min(e->host_m - 1, e->cfg.burnin + e->cfg.iterations) -
                               e->cfg.burnin);
}

int cmc_engine_diagnostics(cmc_engine* e, const cmc_diag_view* o, cmc_error* err) {
  if (!e || !o || !e->begun) {
    set_err(err, CMC_ERR_ARG, "diagnostics need a finished run()");
    return CMC_ERR_ARG;
  }
  if (e->C < 2) return fail_config(err, "gelman_rhat needs at least 2 chains");
  if (e->C > 32) return fail_config(err, "diagnostics support at most 32 chains");
  if (e->split_tail) {
    set_err(err, CMC_ERR_ARG, "diagnostics of a sharded engine: merge the ranks' outputs into an unsharded engine "
                "(cmc_engine_set_output; Python: shards.gather_shard_outputs + load_outputs)");
    return CMC_ERR_ARG;
  }
  const long count = monitored_count(e);
  if (count < 2) return fail_config(err, "gelman_rhat needs at least 2 iterations");
  std::vector<double> vals;
  std::vector<int> flags;
  int rc = diag_to_host(e, count, vals, flags, err);
  if (rc) return rc;
  const long R = 2 + 2 * e->L + e->G * (e->L + 1);
  double* dsts[5] = {o->rhat, o->mean, o->sd, o->ci_lo, o->ci_hi};
  for (int k = 0; k < 5; ++k)
    if (dsts[k]) std::memcpy(dsts[k], vals.data() + (size_t)k * R, sizeof(double) * R);
  if (o->flags) std::memcpy(o->flags, flags.data(), sizeof(int) * R);
  if (o->ess && e->n_cols)
    std::memcpy(o->ess, vals.data() + 5 * R, sizeof(double) * e->n_cols);
  if (o->ess_status && e->n_cols)
    std::memcpy(o->ess_status, flags.data() + R, sizeof(int) * e->n_cols);
  return CMC_OK;
}

// write_results (P:src/io.cpp:571-720): device diagnostics + host writer.
int cmc_engine_write_results(cmc_engine* e, const char* outdir, const char* const* genes,
                             const char* const* contrast_ids, double wall_seconds,
                             cmc_error* err) {
  if (!e || !outdir || !e->begun) {
    set_err(err, CMC_ERR_ARG, "write_results needs a finished run()");
    return CMC_ERR_ARG;
  }
  if (e->split_tail) {
    set_err(err, CMC_ERR_ARG, "write_results of a sharded engine: merge the ranks' outputs into an unsharded engine "
                "(cmc_engine_set_output; Python: shards.gather_shard_outputs + load_outputs)");
    return CMC_ERR_ARG;
  }
  if (e->C > 32) return fail_config(err, "diagnostics support at most 32 chains");
  const long C = e->C, G = e->G, L = e->L;
  const long count = monitored_count(e);
  cmc::ResultsInput in;
  in.outdir = outdir;
  in.C = C;
  in.G = G;
  in.N = e->N;
  in.L = L;
  in.genes = genes;
  in.z = normal_quantile(1.0 - 0.05 / 2.0);
  // build_diagnostics throws for < 2 chains or < 2 iterations (gelman_rhat,
  // P:src/diagnostics.cpp:13-15) after the estimate files are written
  if (C < 2) {
    in.diag_error = true;
    in.diag_error_msg = "gelman_rhat needs at least 2 chains";
  } else if (count < 2) {
    in.diag_error = true;
    in.diag_error_msg = "gelman_rhat needs at least 2 iterations";
  }
  std::vector<double> vals;
  std::vector<int> flags;
  int rc = diag_to_host(e, count, vals, flags, err);
  if (rc) return rc;
  const long R = 2 + 2 * L + G * (L + 1);
  auto part = [&](int k) {
    return std::vector<double>(vals.begin() + (size_t)k * R, vals.begin() + (size_t)(k + 1) * R);
  };
  in.rhat = part(0);
  in.mean = part(1);
  in.sd = part(2);
  in.lo = part(3);
  in.hi = part(4);
  in.flags.assign(flags.begin(), flags.begin() + R);
  in.ess.assign(vals.begin() + 5 * R, vals.end());
  in.ess_status.assign(flags.begin() + R, flags.end());
  // thinned-sample columns (engine.cpp:390-400) and each row's column
  const long nsv = (long)e->saved.size();
  in.col_names = {"nu", "tau"};
  for (long l = 0; l < L; ++l) in.col_names.push_back("theta[" + std::to_string(l + 1) + "]");
  for (long l = 0; l < L; ++l) in.col_names.push_back("sigma[" + std::to_string(l + 1) + "]");
  in.row_col.assign((size_t)R, -1);
  for (long r = 0; r < 2 + 2 * L; ++r) in.row_col[(size_t)r] = r;
  for (long k = 0; k < nsv; ++k) {
    const long g = e->saved[(size_t)k];
    for (long l = 0; l < L; ++l) {
      in.row_col[(size_t)(2 + 2 * L + g * L + l)] = (long)in.col_names.size();
      in.col_names.push_back("beta[" + std::to_string(g + 1) + "," + std::to_string(l + 1) + "]");
    }
    in.row_col[(size_t)(2 + 2 * L + G * L + g)] = (long)in.col_names.size();
    in.col_names.push_back("gamma[" + std::to_string(g + 1) + "]");
  }
  if ((long)in.col_names.size() != e->n_cols) return fail_config(err, "internal: column count");
  // contrasts
  if (e->has_ctab) {
    for (int k = 0; k < e->ctab.n; ++k) {
      in.contrast_ids.push_back(contrast_ids && contrast_ids[k]
                                    ? std::string(contrast_ids[k])
                                    : "contrast" + std::to_string(k + 1));
      in.per_gene.push_back(e->ctab.per_gene[k]);
      in.prob_off.push_back(e->ctab.prob_off[k]);
    }
    in.n_prob = e->ctab.n_prob;
    in.probs.resize((size_t)C * in.n_prob);
    CUDA_TRY(cudaMemcpy(in.probs.data(), e->cprob.p, sizeof(double) * in.probs.size(),
                        cudaMemcpyDeviceToHost));
  }
  // samples: completed rows only
  in.rows = std::min<long>(e->n_rows, count / e->cfg.thin);
  in.samples.resize((size_t)C * e->n_cols * in.rows);
  if (in.rows > 0)
    CUDA_TRY(cudaMemcpy2D(in.samples.data(), sizeof(double) * in.rows, e->samples.p,
                          sizeof(double) * e->n_rows, sizeof(double) * in.rows,
                          (size_t)C * e->n_cols, cudaMemcpyDeviceToHost));
  for (long r = 0; r < in.rows; ++r) in.sample_iters.push_back(e->cfg.burnin + (r + 1) * e->cfg.thin);
  // run report
  in.version = cmc_version();
  in.seed = e->cfg.seed;
  in.chains = e->cfg.chains;
  in.iterations = e->cfg.iterations;
  in.burnin = e->cfg.burnin;
  in.tune_cutoff = e->cfg.tune_cutoff;
  in.thin = e->cfg.thin;
  in.workers = e->cfg.workers;
  in.max_step_out = e->cfg.max_step_out;
  in.save_genes = e->cfg.save_genes;
  in.slice_faithful = e->cfg.sampler_mode == CMC_SLICE_FAITHFUL;
  in.wall_seconds = wall_seconds;
  std::vector<Hyper> hp((size_t)C);
  CUDA_TRY(cudaMemcpy(hp.data(), e->hyper.p, sizeof(Hyper) * C, cudaMemcpyDeviceToHost));
  for (long c = 0; c < C; ++c) {
    // per-step timing mode: the 7 steps; otherwise the fused device sweep
    // under the first step
    std::vector<double> st(7, 0.0);
    if (e->step_timed)
      st.assign(e->step_sec.begin() + c * 7, e->step_sec.begin() + c * 7 + 7);
    else
      st[0] = e->sweep_seconds;
    in.step_seconds.push_back(st);
    in.clamp_events.push_back(hp[(size_t)c].clamps);
  }
  in.saved_genes = e->saved;
  return cmc::write_results_files(in, err);
}

// Debug timeline: record warp start/end times of the next `sweeps` sweeps
// (direct launches on the lanes, no graph); returns the record count.
int cmc_engine_trace(cmc_engine* e, long m_begin, long sweeps, unsigned long long* out,
                     long cap, long* n_out, cmc_error* err) {
  if (!e || !e->begun || sweeps < 1) {
    set_err(err, CMC_ERR_ARG, "trace needs begin()");
    return CMC_ERR_ARG;
  }
  CUDA_TRY(cudaSetDevice(e->device));
  int rc = set_device_m(e, m_begin, err);
  if (rc) return rc;
  unsigned long long* d_tr = nullptr;
  unsigned int* d_n = nullptr;
  CUDA_TRY(cudaMalloc(&d_tr, sizeof(unsigned long long) * 3 * cap));
  CUDA_TRY(cudaMalloc(&d_n, sizeof(unsigned int)));
  CUDA_TRY(cudaMemset(d_n, 0, sizeof(unsigned int)));
  SweepParams p = e->base;
  p.monitor_enabled = 1;
  p.trace = d_tr;
  p.trace_n = d_n;
  p.trace_cap = (unsigned)cap;
  // the traced sweeps replay from one graph, as production sweeps do
  // (eager launches add launch and cross-stream gaps of their own)
  cudaGraph_t gr;
  cudaGraphExec_t ge = nullptr;
  CUDA_TRY(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
  cudaError_t r = fork_lanes(e);
  for (long off = 0; r == cudaSuccess && off < sweeps; ++off) r = enqueue_all_lanes(e, p, off);
  if (r == cudaSuccess) r = join_lanes(e);
  if (r == cudaSuccess) r = launch_advance(e->d_m.p, sweeps, e->stream);
  cudaError_t r2 = cudaStreamEndCapture(e->stream, &gr);
  CUDA_TRY(r);
  CUDA_TRY(r2);
  r = cudaGraphInstantiate(&ge, gr, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(gr);
  CUDA_TRY(r);
  CUDA_TRY(cudaGraphLaunch(ge, e->stream));
  CUDA_TRY(cudaStreamSynchronize(e->stream));
  cudaGraphExecDestroy(ge);
  e->host_m = m_begin + sweeps;
  unsigned int n = 0;
  CUDA_TRY(cudaMemcpy(&n, d_n, sizeof(n), cudaMemcpyDeviceToHost));
  n = std::min<unsigned>(n, (unsigned)cap);
  CUDA_TRY(cudaMemcpy(out, d_tr, sizeof(unsigned long long) * 3 * n, cudaMemcpyDeviceToHost));
  *n_out = n;
  cudaFree(d_tr);
  cudaFree(d_n);
  return CMC_OK;
}

int cmc_engine_get_output(cmc_engine* e, long chain, const cmc_output_view* o,
                          cmc_error* err) {
  if (!e || !o || chain < 0 || chain >= e->C) {
    set_err(err, CMC_ERR_ARG, "bad chain");
    return CMC_ERR_ARG;
  }
  int rc = ensure_device(e, err);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(e->device));
  CUDA_TRY(cudaStreamSynchronize(e->stream));
  const long Gt = e->G_total, G = e->G, N = e->N, L = e->L, g0 = e->g0;
  const size_t so = (size_t)chain;
  Hyper hp;
  CUDA_TRY(cudaMemcpy(&hp, e->hyper.p + chain, sizeof(Hyper), cudaMemcpyDeviceToHost));
  const long count = std::max<long>(0, std::min(e->host_m - 1, e->cfg.burnin + e->cfg.iterations) - e->cfg.burnin);
  if (o->acc_count) *o->acc_count = count;
  double* outs[4] = {o->acc_mean, o->acc_meansq, o->acc_mean_c, o->acc_meansq_c};
  std::vector<double> buf;
  for (int k = 0; k < 4; ++k) {
    double* dst = outs[k];
    if (!dst) continue;
    long i = 0;
    dst[i++] = hp.acc[k][0];
    dst[i++] = hp.acc[k][1];
    for (long l = 0; l < L; ++l) dst[i++] = hp.acc[k][2 + l];
    for (long l = 0; l < L; ++l) dst[i++] = hp.acc[k][2 + L + l];
    // beta G x L, gamma G, eps G x N: device transpose, one copy each
    CUDA_TRY(device_to_aos(e, e->acc_beta.p + so * 4 * L * G + (size_t)k * L * G,
                           dst + i + g0 * L, L));
    i += Gt * L;
    CUDA_TRY(cudaMemcpy(dst + i + g0, e->acc_gam.p + so * 4 * G + (size_t)k * G,
                        sizeof(double) * G, cudaMemcpyDeviceToHost));
    i += Gt;
    CUDA_TRY(device_to_aos(e, e->acc_eps.p + so * 4 * N * G + (size_t)k * N * G,
                           dst + i + g0 * N, N));
    i += Gt * N;
    if (e->xi_any) {
      // xi block (extension): sampled columns from the device; a normal
      // column's xi is the constant 1, whose compensated Welford state after
      // `count` updates is (1, 1, 0, 0)
      CUDA_TRY(device_to_aos(e, e->acc_xi.p + so * 4 * L * G + (size_t)k * L * G,
                             dst + i + g0 * L, L));
      const double konst = (k < 2 && count > 0) ? 1.0 : 0.0;
      for (long l = 0; l < L; ++l)
        if (e->prior[(size_t)l] == CMC_PRIOR_NORMAL)
          for (long g = 0; g < G; ++g) dst[i + (g0 + g) * L + l] = konst;
    }
  }
  if (e->has_ctab) {
    if (o->contrast_prob)
      CUDA_TRY(cudaMemcpy(o->contrast_prob, e->cprob.p + so * e->ctab.n_prob,
                          sizeof(double) * e->ctab.n_prob, cudaMemcpyDeviceToHost));
    if (o->contrast_count)
      for (int ci = 0; ci < e->ctab.n; ++ci) o->contrast_count[ci] = count;
  }
  const long rows = std::min<long>(e->n_rows, count / e->cfg.thin);
  if (o->samples && e->n_cols * e->n_rows > 0) {
    buf.resize((size_t)e->n_cols * e->n_rows);
    CUDA_TRY(cudaMemcpy(buf.data(), e->samples.p + so * e->n_cols * e->n_rows,
                        sizeof(double) * buf.size(), cudaMemcpyDeviceToHost));
    // the reference keeps only completed rows: samples[col].size() == rows
    for (long c = 0; c < e->n_cols; ++c)
      for (long r = 0; r < rows; ++r) o->samples[c * rows + r] = buf[(size_t)c * e->n_rows + r];
  }
  if (o->sample_iters)
    for (long r = 0; r < rows; ++r) o->sample_iters[r] = e->cfg.burnin + (r + 1) * e->cfg.thin;
  if (o->clamp_events) *o->clamp_events = hp.clamps;
  if (o->final_state) {
    if ((rc = download_state(e, chain, o->final_state, nullptr, nullptr, err))) return rc;
  }
  if (o->step_seconds) {
    // per-step timing mode: the 7 steps; otherwise the fused device sweep
    // under the first step
    for (int k = 0; k < 7; ++k)
      o->step_seconds[k] = e->step_timed ? e->step_sec[(size_t)chain * 7 + k] : 0.0;
    if (!e->step_timed) o->step_seconds[0] = e->sweep_seconds;
  }
  return CMC_OK;
}

// The inverse of cmc_engine_get_output, for results of a sharded job: the
// ranks' outputs, merged on the host, are loaded into an unsharded engine
// of the full problem, whose device diagnostics and results writer then
// run as after its own run().
int cmc_engine_set_output(cmc_engine* e, long chain, const cmc_output_view* o,
                          cmc_error* err) {
  if (!e || !o || chain < 0 || chain >= e->C || !o->acc_count || !o->acc_mean ||
      !o->acc_meansq || !o->acc_mean_c || !o->acc_meansq_c) {
    set_err(err, CMC_ERR_ARG, "bad chain or incomplete output view");
    return CMC_ERR_ARG;
  }
  if (e->split_tail) {
    set_err(err, CMC_ERR_ARG, "set_output needs an unsharded engine of the full problem");
    return CMC_ERR_ARG;
  }
  const long count = *o->acc_count;
  if (count < 0 || count > e->cfg.iterations) {
    set_err(err, CMC_ERR_ARG, "monitored count out of range");
    return CMC_ERR_ARG;
  }
  if (e->begun && chain > 0 && monitored_count(e) != count) {
    set_err(err, CMC_ERR_ARG, "every chain needs the same monitored count");
    return CMC_ERR_ARG;
  }
  int rc = ensure_device(e, err);
  if (rc) return rc;
  CUDA_TRY(cudaSetDevice(e->device));
  const long G = e->G, N = e->N, L = e->L;
  const size_t so = (size_t)chain;
  if (o->final_state && (rc = upload_state(e, chain, o->final_state, nullptr, nullptr, err)))
    return rc;
  CUDA_TRY(cudaStreamSynchronize(e->stream));
  Hyper hp;
  CUDA_TRY(cudaMemcpy(&hp, e->hyper.p + chain, sizeof(Hyper), cudaMemcpyDeviceToHost));
  const double* src[4] = {o->acc_mean, o->acc_meansq, o->acc_mean_c, o->acc_meansq_c};
  for (int k = 0; k < 4; ++k) {
    const double* a = src[k];
    long i = 0;
    hp.acc[k][0] = a[i++];
    hp.acc[k][1] = a[i++];
    for (long l = 0; l < 2 * L; ++l) hp.acc[k][2 + l] = a[i++];
    CUDA_TRY(aos_to_device(e, a + i, e->acc_beta.p + so * 4 * L * G + (size_t)k * L * G, L));
    i += G * L;
    CUDA_TRY(cudaMemcpyAsync(e->acc_gam.p + so * 4 * G + (size_t)k * G, a + i,
                             sizeof(double) * G, cudaMemcpyHostToDevice, e->stream));
    i += G;
    CUDA_TRY(aos_to_device(e, a + i, e->acc_eps.p + so * 4 * N * G + (size_t)k * N * G, N));
    i += G * N;
    if (e->xi_any)
      CUDA_TRY(aos_to_device(e, a + i, e->acc_xi.p + so * 4 * L * G + (size_t)k * L * G, L));
  }
  if (o->clamp_events) hp.clamps = *o->clamp_events;
  hp.err_key = kNoError;
  hp.err_key_eps = kNoError;
  CUDA_TRY(cudaMemcpyAsync(e->hyper.p + chain, &hp, sizeof(Hyper), cudaMemcpyHostToDevice,
                           e->stream));
  if (e->has_ctab && o->contrast_prob)
    CUDA_TRY(cudaMemcpyAsync(e->cprob.p + so * e->ctab.n_prob, o->contrast_prob,
                             sizeof(double) * e->ctab.n_prob, cudaMemcpyHostToDevice, e->stream));
  if (e->n_cols * e->n_rows > 0) {
    // host [col][rows] (completed rows only) -> device [col][n_rows]
    const long rows = std::min<long>(e->n_rows, count / e->cfg.thin);
    std::vector<double> buf((size_t)e->n_cols * e->n_rows, 0.0);
    if (o->samples)
      for (long c = 0; c < e->n_cols; ++c)
        for (long r = 0; r < rows; ++r) buf[(size_t)c * e->n_rows + r] = o->samples[c * rows + r];
    CUDA_TRY(cudaMemcpyAsync(e->samples.p + so * e->n_cols * e->n_rows, buf.data(),
                             sizeof(double) * buf.size(), cudaMemcpyHostToDevice, e->stream));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(e->stream));
  e->host_m = e->cfg.burnin + count + 1;  // monitored_count() == count
  e->begun = true;
  return CMC_OK;
}

int cmc_nccl_unique_id(void* out128, cmc_error* err) {
  std::string why;
  if (!g_nccl.load(why)) {
    set_err(err, CMC_ERR_NCCL, why);
    return CMC_ERR_NCCL;
  }
  nccl_uid id;
  if (g_nccl.get_uid(&id) != 0) {
    set_err(err, CMC_ERR_NCCL, "ncclGetUniqueId failed");
    return CMC_ERR_NCCL;
  }
  std::memcpy(out128, &id, sizeof(id));
  return CMC_OK;
}

int cmc_engine_shard(cmc_engine* e, int rank, int world, const void* uid,
                     cmc_error* err) {
  if (!e || world < 1 || rank < 0 || rank >= world) {
    set_err(err, CMC_ERR_ARG, "bad rank/world");
    return CMC_ERR_ARG;
  }
  if (e->dev_ready) {
    set_err(err, CMC_ERR_ARG, "cmc_engine_shard must precede device use");
    return CMC_ERR_ARG;
  }
  long b = 0, en = 0;
  cmc_shard_bounds(e->G_total, rank, world, &b, &en);
  if (en <= b) {
    set_err(err, CMC_ERR_CONFIG, "shard has no genes: use fewer ranks for this G");
    return CMC_ERR_CONFIG;
  }
  if (e->loop) {
    set_err(err, CMC_ERR_ARG, "engine already joined a loopback group");
    return CMC_ERR_ARG;
  }
  e->rank = rank;
  e->world = world;
  e->g0 = b;
  e->G = en - b;
  // world == 1 with an id still builds a (1-rank) clique: the exchange path
  // then runs on one GPU, which is how it is tested without a second GPU
  if (world > 1 || uid) {
    std::string why;
    if (!g_nccl.load(why)) {
      set_err(err, CMC_ERR_NCCL, why);
      return CMC_ERR_NCCL;
    }
    CUDA_TRY(cudaSetDevice(e->device));
    nccl_uid id;
    std::memcpy(&id, uid, sizeof(id));
    if (g_nccl.init_rank(&e->comm, world, id, rank) != 0) {
      set_err(err, CMC_ERR_NCCL, "ncclCommInitRank failed");
      return CMC_ERR_NCCL;
    }
    e->split_tail = true;
    // chain lanes: one split communicator per extra lane (collective; every
    // rank has the same chain count, hence the same lane count)
    e->split_lanes = 1;
    const int want = (int)std::min<long>(e->C, CMC_MAX_LANES);
    if (want > 1 && g_nccl.comm_split) {
      int k = 1;
      for (; k < want; ++k)
        if (g_nccl.comm_split(e->comm, 0, rank, &e->lane_comm[k], nullptr) != 0) break;
      e->split_lanes = k;
    }
  }
  return CMC_OK;
}

int cmc_loopback_create(int world, cmc_loopback** out, cmc_error* err) {
  if (world < 1 || !out) {
    set_err(err, CMC_ERR_ARG, "bad world or output pointer");
    return CMC_ERR_ARG;
  }
  cmc_loopback* g = new cmc_loopback;
  g->world = world;
  g->send.assign((size_t)world, nullptr);
  g->ready.assign((size_t)world, nullptr);
  g->copied.assign((size_t)world, nullptr);
  *out = g;
  return CMC_OK;
}

int cmc_loopback_destroy(cmc_loopback* g) {
  delete g;
  return CMC_OK;
}

int cmc_engine_shard_loopback(cmc_engine* e, int rank, cmc_loopback* g, cmc_error* err) {
  if (!e || !g || rank < 0 || rank >= g->world) {
    set_err(err, CMC_ERR_ARG, "bad rank or loopback group");
    return CMC_ERR_ARG;
  }
  if (e->dev_ready || e->comm || e->loop) {
    set_err(err, CMC_ERR_ARG, "cmc_engine_shard_loopback must precede device use and sharding");
    return CMC_ERR_ARG;
  }
  long b = 0, en = 0;
  cmc_shard_bounds(e->G_total, rank, g->world, &b, &en);
  if (en <= b) {
    set_err(err, CMC_ERR_CONFIG, "shard has no genes: use fewer ranks for this G");
    return CMC_ERR_CONFIG;
  }
  CUDA_TRY(cudaSetDevice(e->device));
  CUDA_TRY(cudaEventCreateWithFlags(&e->loop_ready, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&e->loop_copied, cudaEventDisableTiming));
  e->rank = rank;
  e->world = g->world;
  e->g0 = b;
  e->G = en - b;
  e->loop = g;
  e->split_tail = true;
  e->split_lanes = 1;
  return CMC_OK;
}

// ------------------------------------------------------- synthetic inputs

namespace {
// The reference draws counts with std::poisson_distribution<long long> over
// its RngStream (P:src/simulate.cpp:82-83); Stream is the same Philox
// stream, so the same standard-library distribution over it gives the
// reference's counts bit for bit (same libstdc++ and glibc libm).
struct StreamUrbg {
  using result_type = uint64_t;
  Stream* s;
  static constexpr result_type min() { return 0; }
  static constexpr result_type max() { return ~0ull; }
  result_type operator()() { return s->next(); }
};
}  // namespace

int cmc_simulate(long G, long N, long L, const double* X, const double* h,
                 double nu, double tau, const double* theta,
                 const double* sigma, uint64_t seed, long long* counts,
                 cmc_error* err) {
  if (G < 1 || N < 1 || L < 1 || !X || !theta || !sigma || !counts) {
    set_err(err, CMC_ERR_ARG, "bad simulation arguments");
    return CMC_ERR_ARG;
  }
  if (!(nu > 0.0) || !(tau > 0.0)) {
    set_err(err, CMC_ERR_CONFIG, "nu and tau must be positive");
    return CMC_ERR_CONFIG;
  }
  std::vector<double> beta((size_t)L);
  for (long g = 0; g < G; ++g) {
    // beta, gamma, eps draws as P:src/simulate.cpp:51-69
    Stream rng;
    rng.init(seed, 0, 0, site_id(kSiteSim, (uint64_t)g));
    for (long l = 0; l < L; ++l) beta[l] = theta[l] + sigma[l] * normal(rng);
    const double gam = 1.0 / gamma_draw(rng, nu / 2.0, nu * tau / 2.0);
    const double sd = std::sqrt(gam);
    for (long n = 0; n < N; ++n) {
      const double e = sd * normal(rng);
      double eta = 0.0;
      for (long l = 0; l < L; ++l) eta += X[n * L + l] * beta[l];
      const double arg = (h ? h[n] : 0.0) + e + eta;
      // SimulationError cases, P:src/simulate.cpp:64-81
      if (arg > 700.0) {
        char buf[160];
        std::snprintf(buf, sizeof(buf),
                      "simulated Poisson mean overflow at gene %ld, sample %ld "
                      "(log mean %.6g exceeds %.0f)",
                      g + 1, n + 1, arg, 700.0);
        set_err(err, CMC_ERR_CONFIG, buf);
        return CMC_ERR_CONFIG;
      }
      const double lambda = std::exp(arg);
      if (lambda > 1e15) {
        char buf[160];
        std::snprintf(buf, sizeof(buf),
                      "simulated Poisson mean %.6g at gene %ld, sample %ld is "
                      "too large for integer counts",
                      lambda, g + 1, n + 1);
        set_err(err, CMC_ERR_CONFIG, buf);
        return CMC_ERR_CONFIG;
      }
      std::poisson_distribution<long long> pois(lambda);
      StreamUrbg u{&rng};
      counts[g * N + n] = pois(u);
    }
  }
  return CMC_OK;
}

}  // extern "C"
