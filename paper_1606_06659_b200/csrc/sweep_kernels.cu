// B200 kernels for one Gibbs sweep of the two-level Poisson-lognormal model
// (reference GibbsEngine::iterate, P:src/engine.cpp:161-370, plus the
// run_chain monitors, P:src/engine.cpp:409-447).
//
// Per iteration m and chain lane (single GPU, captured in CUDA graphs):
//   eps_sweep   one thread per (gene, sample): eps_gn (step 1) and its
//               Welford monitor.
//   gene_sweep  one thread per gene: gamma_g (step 2), beta_g1..beta_gL
//               (step 5), their monitors, per-gene contrasts, thinning; the
//               last of a 1024-gene leaf's blocks sums the leaf (log gamma,
//               1/gamma, beta_l: the reference tree's leaves,
//               P:include/countmc/parallel.hpp:67-84).
//   hyper_a     one block per chain: pairwise sums over the leaves, nu, tau
//               (steps 3-4) and theta (step 6).
//   leaf_b      leaf sums of (beta_l - theta_l)^2; the last block draws
//               sigma (step 7) and updates the hyper monitors / thinning.
// With a xi prior the xi kernel follows the gene kernel and leaf_a (its
// last block running steps 3, 4, 6) replaces the fused leaf sums.
// Multi-GPU sums local leaves, all-gathers the partial sums (with each
// rank's stall flag), and runs hyper_a / hyper_b as single-block kernels.
//
// Compiled with -fmad=false: every expression below rounds exactly as the
// reference's non-FMA x86-64 build (P:CMakeLists.txt:7-9), which makes the
// sampled values bit-identical to the reference for identical uniforms.
#include <math.h>

#include "fastmath.cuh"
#include "rng.cuh"
#include <algorithm>
#include <cassert>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "sweep.h"

namespace cmc {

namespace {

constexpr double kExpClamp = 700.0;  // P:include/countmc/model.hpp:14

struct SliceCfg {
  int K;
  int max_shrink;
  long burnin;
  long tune_cutoff;
  uint64_t reject_below;  // 2^64 mod (K+1)
  uint64_t inv;           // floor(2^64 / (K+1))
};

// P:include/countmc/slice.hpp:27-35
__device__ __forceinline__ void tune_update(double& w, double& wa, long m,
                                            double delta, long cutoff) {
  const double md = (double)m;
  wa += md * delta;
  if (m > cutoff) {
    const double nw = wa / (0.5 * md * (md + 1.0));
    if (nw >= 1e-12) w = nw;
  }
}

// Stepping-out + shrinkage slice step with the reference's draw order
// (P:include/countmc/slice.hpp:42-75), written as ONE loop that performs
// one log-density evaluation per trip whatever phase (step-out left,
// step-out right, shrink) a lane is in: a warp pays the maximum of the
// lanes' total evaluation counts, not the sum of per-phase maxima.  The
// trip body is branch-free (each lane computes every phase's update and
// keeps the one its phase selects), so diverged lanes still issue as one
// SIMT stream; only the rare refill of a third Philox block branches.
template <class F, class RNG = Stream>
__device__ __forceinline__ double slice_step(F& f, double x0, double& w,
                                             double& wa, const SliceCfg& sc,
                                             long m, RNG& rng,
                                             bool& stalled) {
  const double fx0 = f(x0);
  const double logu = fx0 + log(rng.u01());
  const double wv = w;
  double lo = x0 - wv * rng.u01();
  double hi = lo + wv;
  const int kl0 = (int)rng.uniform_int_pre((uint64_t)sc.K + 1, sc.reject_below, sc.inv);
  int kl = kl0, kr = sc.K - kl0;
  int phase = kl > 0 ? 0 : (kr > 0 ? 1 : 2);
  int it = 0;
  double x1 = x0;
  for (;;) {
    const bool S = phase == 2;
    if (S && rng.na == 0) rng.refill();
    const double u = ((double)(rng.a0 >> 11) + 0.5) * 0x1.0p-53;
    if (S) {  // pop (predicated moves)
      rng.a0 = rng.a1;
      rng.a1 = rng.a2;
      rng.a2 = rng.a3;
      --rng.na;
    }
    const double xs = lo + (hi - lo) * u;
    const double xe = S ? xs : (phase == 0 ? lo : hi);
    const double fe = f(xe);
    const bool Lp = phase == 0, Rp = phase == 1;
    const bool in = logu < fe;
    const bool acc = S && (fe > logu);
    const bool rej = S && !(fe > logu);
    lo = (Lp && in) ? lo - wv : lo;
    hi = (Rp && in) ? hi + wv : hi;
    kl -= (Lp && in) ? 1 : 0;
    kr -= (Rp && in) ? 1 : 0;
    hi = (rej && xs > x0) ? xs : hi;
    lo = (rej && !(xs > x0)) ? xs : lo;
    it += rej ? 1 : 0;
    x1 = S ? xs : x1;
    const int after_l = kr > 0 ? 1 : 2;
    phase = (Lp && !(in && kl > 0)) ? after_l : ((Rp && !(in && kr > 0)) ? 2 : phase);
    if (acc) break;
    if (it >= sc.max_shrink) {
      stalled = true;
      return x0;
    }
  }
  if (m <= sc.burnin) tune_update(w, wa, m, fabs(x1 - x0), sc.tune_cutoff);
  return x1;
}

// slice_step as a resumable state machine (same draws, same evaluation
// order, same trip body): start() draws log u, the placement and K_L;
// trips() runs at most `max_trips` trips and reports running / accepted /
// stalled; finish() applies the tuning update.  A lane's whole state
// (SliceRun + the Stream queue) can be parked in shared memory after a
// bounded first pass and resumed by another thread (xi_sweep_kernel).
struct SliceRun {
  double x0, logu, lo, hi, x1, wv;
  int kl, kr, phase, it;
};
enum : int { kSliceRunning = 0, kSliceAccepted = 1, kSliceStalled = 2 };

template <class F>
__device__ __forceinline__ void slice_start(F& f, double x0, double w, const SliceCfg& sc,
                                            Stream& rng, SliceRun& s) {
  const double fx0 = f(x0);
  s.x0 = x0;
  s.logu = fx0 + log(rng.u01());
  s.wv = w;
  s.lo = x0 - w * rng.u01();
  s.hi = s.lo + w;
  const int kl0 = (int)rng.uniform_int_pre((uint64_t)sc.K + 1, sc.reject_below, sc.inv);
  s.kl = kl0;
  s.kr = sc.K - kl0;
  s.phase = s.kl > 0 ? 0 : (s.kr > 0 ? 1 : 2);
  s.it = 0;
  s.x1 = x0;
}

template <class F>
__device__ __forceinline__ int slice_trips(F& f, const SliceCfg& sc, Stream& rng, SliceRun& s,
                                           int max_trips) {
  double lo = s.lo, hi = s.hi, x1 = s.x1;
  int kl = s.kl, kr = s.kr, phase = s.phase, it = s.it;
  const double wv = s.wv, logu = s.logu, x0 = s.x0;
  int res = kSliceRunning;
  for (int trip = 0; trip < max_trips; ++trip) {
    const bool S = phase == 2;
    if (S && rng.na == 0) rng.refill();
    const double u = ((double)(rng.a0 >> 11) + 0.5) * 0x1.0p-53;
    if (S) {
      rng.a0 = rng.a1;
      rng.a1 = rng.a2;
      rng.a2 = rng.a3;
      --rng.na;
    }
    const double xs = lo + (hi - lo) * u;
    const double xe = S ? xs : (phase == 0 ? lo : hi);
    const double fe = f(xe);
    const bool Lp = phase == 0, Rp = phase == 1;
    const bool in = logu < fe;
    const bool acc = S && (fe > logu);
    const bool rej = S && !(fe > logu);
    lo = (Lp && in) ? lo - wv : lo;
    hi = (Rp && in) ? hi + wv : hi;
    kl -= (Lp && in) ? 1 : 0;
    kr -= (Rp && in) ? 1 : 0;
    hi = (rej && xs > x0) ? xs : hi;
    lo = (rej && !(xs > x0)) ? xs : lo;
    it += rej ? 1 : 0;
    x1 = S ? xs : x1;
    const int after_l = kr > 0 ? 1 : 2;
    phase = (Lp && !(in && kl > 0)) ? after_l : ((Rp && !(in && kr > 0)) ? 2 : phase);
    if (acc) {
      res = kSliceAccepted;
      break;
    }
    if (it >= sc.max_shrink) {
      res = kSliceStalled;
      break;
    }
  }
  s.lo = lo;
  s.hi = hi;
  s.x1 = x1;
  s.kl = kl;
  s.kr = kr;
  s.phase = phase;
  s.it = it;
  return res;
}

// Two-phase slice step for log densities whose exp terms are exp(v x + c):
// the step-out evaluation points move by exactly -w (left) / +w (right)
// and the step-out draws no random numbers, so (1) both sides step out in
// the same trip -- the reference runs left then right, but each side's
// stopping rule depends only on its own evaluations -- and (2) each side
// carries exp(v x + c) multiplicatively (times exp(-/+ v w)) instead of
// recomputing it.  The evaluation points lo, hi themselves are updated
// exactly as the reference does (lo -= w, hi += w), so the slice result is
// unchanged; the multiplicative exp differs from a fresh exp in the last
// bits only, which decides comparisons like libm differences do.  Clamp
// events are counted only for evaluations the reference performs.  The
// shrinkage phase uses the full density.  F provides operator() (full),
// side_init(lo, hi, w), any_fresh(), eval_l/eval_r<FRESH>(x, counted) and
// step_l/step_r().
template <class F, class RNG>
__device__ __forceinline__ double slice_step_so2(F& f, double x0, double& w,
                                                 double& wa, const SliceCfg& sc,
                                                 long m, RNG& rng,
                                                 bool& stalled) {
  const double fx0 = f(x0);
  const double logu = fx0 + log(rng.u01());
  const double wv = w;
  double lo = x0 - wv * rng.u01();
  double hi = lo + wv;
  const int kl0 = (int)rng.uniform_int_pre((uint64_t)sc.K + 1, sc.reject_below, sc.inv);
  int kl = kl0, kr = sc.K - kl0;
  bool goL = kl > 0, goR = kr > 0;
  f.side_init(lo, hi, wv);
  // FRESH: the loop body that can take a fresh exp per side (F::side_init
  // decides); the common case runs a body without any exp.
  auto step_out = [&](auto fresh_tag) {
    constexpr bool FRESH = decltype(fresh_tag)::value;
    while (goL || goR) {
      const double fl = f.template eval_l<FRESH>(lo, goL);
      const double fr = f.template eval_r<FRESH>(hi, goR);
      const bool inL = goL && logu < fl;
      const bool inR = goR && logu < fr;
      if (inL) {
        lo -= wv;
        f.step_l();
      }
      if (inR) {
        hi += wv;
        f.step_r();
      }
      kl -= inL ? 1 : 0;
      kr -= inR ? 1 : 0;
      goL = inL && kl > 0;
      goR = inR && kr > 0;
    }
  };
  if (f.any_fresh())
    step_out(std::true_type{});
  else
    step_out(std::false_type{});
  for (int it = 0;;) {
    const double xs = lo + (hi - lo) * rng.u01();
    if (f(xs) > logu) {
      if (m <= sc.burnin) tune_update(w, wa, m, fabs(xs - x0), sc.tune_cutoff);
      return xs;
    }
    if (xs > x0)
      hi = xs;
    else
      lo = xs;
    if (++it >= sc.max_shrink) {
      stalled = true;
      return x0;
    }
  }
}

// log full conditional of eps_gn, P:src/model.cpp:70-74 (clamped_exp
// :13-19): y*e - exp(min(h + eta + e, 700)) - e*e / (2 gamma).
struct EpsF {
  double y, cn, inv_two_gam, e700;
  ExpTab tab;
  unsigned clamps;
  double EL, ER, rL, rR;  // step-out: exp(cn + lo), exp(cn + hi), exp(-w), exp(w)
  bool fL, fR;            // side evaluates fresh exps (see side_init)
  __device__ __forceinline__ double operator()(double x) {
    const double t = cn + x;
    double e;
    if (t > kExpClamp) {
      ++clamps;
      e = e700;
    } else {
      e = fast_exp_le700(t, tab);
    }
    return y * x - e - x * x * inv_two_gam;
  }
  __device__ __forceinline__ void side_init(double lo, double hi, double w) {
    const double tl = cn + lo, th = cn + hi;
    EL = tl > kExpClamp ? 0.0 : fast_exp_le700(tl, tab);
    rR = fast_exp_le700(fmin(w, kExpClamp), tab);
    rL = 1.0 / rR;
    // hi = lo + w: from a normal EL (and w <= 700) ER is one carried step,
    // the same product the step-out loop forms (no third exp per step)
    if (th > kExpClamp)
      ER = 0.0;
    else if (EL > 1e-290 && w <= kExpClamp)
      ER = EL * rR;
    else
      ER = fast_exp_le700(th, tab);
    // A side carries E multiplicatively only from a normal start (E above
    // 1e-290) and with steps within fast_exp_le700's range (w <= 700).
    // Otherwise -- a side that starts clamped (E = 0 here) or underflowed,
    // or w > 700 -- it evaluates a fresh exp on every unclamped trip, as
    // the reference does.  From a normal start the carried E stays valid:
    // on the right t grows and E is read only while t <= 700 (E <= e^700 <
    // DBL_MAX); on the left E only shrinks, and once below the normal range
    // it is far below the last bit of y x - x^2 / (2 gamma).
    const bool wide = !(w <= kExpClamp);
    fL = wide || !(EL > 1e-290);
    fR = wide || !(ER > 1e-290);
  }
  // Step-out evaluation at x with the carried exp E (or a fresh one, see
  // side_init).  The mode is decided once per side: a per-trip range test
  // on E measured 0.5-2.5% of the sweep.
  template <bool FRESH>
  __device__ __forceinline__ double side_eval(double x, double& E, bool fresh, bool counted) {
    const double t = cn + x;
    const bool cl = t > kExpClamp;
    if (FRESH && fresh && !cl) E = fast_exp_le700(t, tab);
    clamps += (cl && counted) ? 1u : 0u;
    return y * x - (cl ? e700 : E) - x * x * inv_two_gam;
  }
  template <bool FRESH>
  __device__ __forceinline__ double eval_l(double x, bool c) {
    return side_eval<FRESH>(x, EL, fL, c);
  }
  template <bool FRESH>
  __device__ __forceinline__ double eval_r(double x, bool c) {
    return side_eval<FRESH>(x, ER, fR, c);
  }
  __device__ __forceinline__ bool any_fresh() const { return fL || fR; }
  __device__ __forceinline__ void step_l() { EL *= rL; }
  __device__ __forceinline__ void step_r() { ER *= rR; }
};

// log inverse-gamma, P:src/model.cpp:84-87
struct InvGammaF {
  double neg_shape1, scale;
  __device__ __forceinline__ double operator()(double x) const {
    if (!(x > 0.0)) return -INFINITY;
    return neg_shape1 * log(x) - scale / x;
  }
};

// log gamma with rate, P:src/model.cpp:89-92
struct GammaRateF {
  double shape1, rate;
  __device__ __forceinline__ double operator()(double x) const {
    if (!(x > 0.0)) return -INFINITY;
    return shape1 * log(x) - rate * x;
  }
};

// P:src/model.cpp:94-100
struct NuF {
  double Gd, tau, s1, s2, d;
  __device__ __forceinline__ double operator()(double nu) const {
    if (!(nu > 0.0) || !(nu < d)) return -INFINITY;
    return -Gd * lgamma(nu / 2.0) + (Gd * nu / 2.0) * log(nu * tau / 2.0) -
           (nu / 2.0) * (s1 + tau * s2);
  }
};

// P:src/model.cpp:131-136
struct SigmaF {
  double Gd, ss, bound;
  __device__ __forceinline__ double operator()(double s) const {
    if (!(s > 0.0) || !(s < bound)) return -INFINITY;
    return -Gd * log(s) - ss / (2.0 * s * s);
  }
};

// Grouped beta density, P:src/engine.cpp:303-316: exp(base + v b) is
// factored as S_j exp(v_j b) over the distinct nonzero column values.
struct BetaF {
  double a, theta, inv_two_sig2, e700;
  const double* val;   // group values (uniform across the warp)
  const double* S;     // shared memory, stride kGeneThreads
  const double* logS;
  ExpTab tab;
  int J;
  unsigned clamps;
  __device__ __forceinline__ double operator()(double b) {
    double tot = a * b;
    for (int j = 0; j < J; ++j) {
      const double t = val[j] * b;
      const double lS = logS[j * kGeneThreads];
      const double Sj = S[j * kGeneThreads];
      if (lS + t > kExpClamp) {
        ++clamps;
        tot -= e700;
      } else if (Sj > 0.0) {
        tot -= Sj * fast_exp(t, tab);
      }
    }
    const double zz = b - theta;
    return tot - zz * zz * inv_two_sig2;
  }
};

// xi full conditional (extension, no reference: parity unpinned), the
// oracle's orc_log_fc_xi: q = (beta - theta)^2 / (2 sigma^2),
//   laplace   -log(x)/2 - q/x - x/2
//   t(k)      -(k/2 + 3/2) log(x) - (q + k/2)/x
//   horseshoe -log(x) - q/x - log1p(x), evaluated as -log(x (1 + x)) - q/x
//             (one log) below 1e150, as the oracle does
struct XiF {
  int fam;
  double q, k;
  __device__ __forceinline__ double operator()(double x) const {
    if (!(x > 0.0)) return -INFINITY;
    if (fam == CMC_PRIOR_LAPLACE) return -0.5 * log(x) - q / x - 0.5 * x;
    if (fam == CMC_PRIOR_T) return -(0.5 * k + 1.5) * log(x) - (q + 0.5 * k) / x;
    return x < 1e150 ? -log(x * (1.0 + x)) - q / x : -log(x) - q / x - log1p(x);
  }
};

// BetaF with the (at most JR) group sums in registers: same terms in the
// same order; each term is branch-free (the clamp and S_j = 0 cases select
// their value), which keeps the slice loop's evaluation straight-line.
template <int JR>
struct BetaFR {
  double a, theta, inv_two_sig2, e700;
  double v[JR], S[JR], lS[JR];
  ExpTab tab;
  int J;
  unsigned clamps;
  __device__ __forceinline__ double operator()(double b) {
    double tot = a * b;
#pragma unroll
    for (int j = 0; j < JR; ++j) {
      if (j < J) {
        const double t = v[j] * b;
        const bool cl = lS[j] + t > kExpClamp;
        const double e = fast_exp(t, tab);
        clamps += cl ? 1u : 0u;
        tot -= cl ? e700 : (S[j] > 0.0 ? S[j] * e : 0.0);
      }
    }
    const double zz = b - theta;
    return tot - zz * zz * inv_two_sig2;
  }
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Warp timeline record (only when p.trace is set): lane 0 opens a record
// {kernel<<56 | slot<<48 | smid<<32 | blockIdx.x, t_start, t_end} at kernel
// entry, and every lane raises t_end when it leaves (destructor, so every
// return path is covered).
struct WarpTrace {
  unsigned long long* rec;
  __device__ __forceinline__ WarpTrace(const SweepParams& p, int kernel, int slot) : rec(nullptr) {
    if (!p.trace) return;
    unsigned i = 0;
    if ((threadIdx.x & 31) == 0) {
      i = atomicAdd(p.trace_n, 1u);
      if (i < p.trace_cap) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.trace[3 * i] = ((unsigned long long)kernel << 56) |
                         ((unsigned long long)slot << 48) |
                         ((unsigned long long)smid << 32) | blockIdx.x;
        p.trace[3 * i + 1] = gtimer();
        p.trace[3 * i + 2] = 0;
      }
    }
    i = __shfl_sync(__activemask(), i, 0);
    if (i < p.trace_cap) rec = p.trace + 3 * i;
  }
  __device__ __forceinline__ ~WarpTrace() {
    if (rec) atomicMax(rec + 2, gtimer());
  }
};

// Kahan add, P:include/countmc/streaming.hpp:29-34
__device__ __forceinline__ void kahan(double& sum, double& comp, double term) {
  const double y = term - comp;
  const double t = sum + y;
  comp = (t - sum) - y;
  sum = t;
}

// MomentAccumulator::update on SoA storage acc[k * stride] (k = mean,
// meansq, mean_c, meansq_c), P:include/countmc/streaming.hpp:17-22.
__device__ __forceinline__ void moments(double* acc, size_t stride, double v,
                                        double mcount) {
  double mean = acc[0], meansq = acc[stride], mc = acc[2 * stride],
         msc = acc[3 * stride];
  kahan(mean, mc, (v - mean) / mcount);
  kahan(meansq, msc, (v * v - meansq) / mcount);
  acc[0] = mean;
  acc[stride] = meansq;
  acc[2 * stride] = mc;
  acc[3 * stride] = msc;
}

// Every stall of a chain recorded in one slot happens in one iteration
// (later kernels of a stalled chain return at entry), so err_m is written
// with one value.  The eps kernel uses the second slot (err_key_eps): it
// may overlap the previous iteration's tail; the host reports the record
// with the smaller (iteration, key).
__device__ __forceinline__ bool stalled_chain(const Hyper* hp) {
  return hp->err_key != kNoError || hp->err_key_eps != kNoError || hp->peer_stall;
}

// The same test for the tail of iteration m (leaf sums, hyper draws): the
// eps kernel of iteration m + 1 runs beside it, and its stall must not stop
// iteration m's tail (the reference draws nu..sigma of m before eps of
// m + 1).  The eps kernel writes err_m_eps before its key (release), so a
// key seen here has its iteration readable after a fence.
__device__ __forceinline__ bool tail_stalled(const Hyper* hp, long m) {
  if (hp->err_key != kNoError || hp->peer_stall) return true;
  if (*(volatile const unsigned long long*)&hp->err_key_eps == kNoError) return false;
  __threadfence();
  return *(volatile const long long*)&hp->err_m_eps <= m;
}

__device__ __forceinline__ void record_stall(Hyper* hp, unsigned long long key,
                                             long m) {
  atomicMin(&hp->err_key, key);
  hp->err_m = m;
}

// Accessor for the gathered leaf partials of one lane:
// [rank][C][Q][leaves_per_rank], chain index relative to the lane.  Plain
// scalars, not the SweepParams: a reference to the kernel's parameter
// block inside the noinline recursion below would copy the whole block to
// the stack.
struct PartView {
  const double* part;
  long C, c, Q, lpr;  // lane chains, this chain (relative), quantities, leaves/rank
};
__device__ __forceinline__ PartView part_view(const double* part, const SweepParams& p,
                                              int slot, int Q) {
  return PartView{part, p.C, slot - p.slot_base, Q, p.leaves_per_rank};
}
__device__ __forceinline__ double leaf_part(const PartView& v, int q, long leaf) {
  // leaf counts fit 32 bits (< 2^22 leaves at G < 2^32): a 32-bit division
  // (round 1's 64-bit one was a ~100-instruction subroutine call per leaf)
  const unsigned lpr = (unsigned)v.lpr;
  const long r = (unsigned)leaf / lpr, j = (unsigned)leaf - (unsigned)r * lpr;
#ifdef CMC_DEBUG_BOUNDS
  assert(v.c >= 0 && v.c < v.C && q < v.Q);
#endif
  return __ldcg(v.part + (((r * v.C + v.c) * v.Q + q) * v.lpr + j));
}

// pairwise_sum over the leaf partials, P:src/parallel.cpp:81-86.
__device__ __noinline__ double pairwise_leaves(const PartView v, int q, long lo, long n) {
  if (n == 0) return 0.0;
  if (n == 1) return leaf_part(v, q, lo);
  const long mid = n / 2;
  return pairwise_leaves(v, q, lo, mid) + pairwise_leaves(v, q, lo + mid, n - mid);
}

__device__ double param_value(const ContrastTable* t, int k, const double* beta,
                              size_t G, long gl, double gam, const Hyper* hp) {
  const int fam = t->fam[k], idx = t->idx[k];
  switch (fam) {
    case 0: return beta[(size_t)idx * G + gl];
    case 1: return gam;
    case 2: return hp->theta[idx];
    case 3: return hp->sigma[idx];
    case 4: return hp->nu;
    default: return hp->tau;
  }
}

// ContrastAccumulator::update for one slot, P:src/streaming.cpp:90-108.
__device__ void contrast_update(const ContrastTable* t, int ci, double* prob,
                                double mcount, const double* beta, size_t G,
                                long gl, double gam, const Hyper* hp) {
  bool all = true;
  for (int term = t->term_begin[ci]; term < t->term_begin[ci + 1]; ++term) {
    double lhs = 0.0;
    for (int k = t->coef_begin[term]; k < t->coef_begin[term + 1]; ++k)
      lhs += t->coef[k] * param_value(t, k, beta, G, gl, gam, hp);
    if (!(lhs > t->threshold[term])) {
      all = false;
      break;
    }
  }
  const double ind = all ? 1.0 : 0.0;
  *prob += (ind - *prob) / mcount;
}

// ---------------------------------------------------------------- kernels

// Step 1, one thread per (gene, sample): eps_gn are conditionally
// independent given the gene's previous beta and gamma (P:src/engine.cpp:
// 178-202), so the 16 slice steps of a gene run on 16 threads.  A warp holds
// 32 consecutive genes at one sample n (coalesced SoA loads), the grid's y
// dimension is n and z the chain.  The step is latency-bound, so the block
// count per SM is tuned against spills (earlier A/B on B200: 6 blocks 4.18e8, 8 blocks 4.31e8
// gene-iter/s, 9-10 blocks no better once the gene kernel also runs at 6).
// Since the one-decision step-out and the post-step re-convergence, 7
// blocks (72 registers, no spill) edge out 8 (64 registers, 16-byte
// spill): 0.3330 vs 0.3338 ms per 4-chain sweep, 0.133 vs 0.136 ms at 1
// chain (A/B, two reps each).
// r02: with the Philox queue's second block in shared memory, 8 blocks (64
// registers, no spill): 0.3261 vs 0.3281 ms per 4-chain sweep (A/B).
// r02, after the carried beta exps: 9 blocks (56 registers) with the gene
// kernel at 5: 0.3268 vs 0.3290 ms (100-sweep calls), 0.3316 vs 0.3330
// (20-sweep calls), two reps on two boxes; 10 blocks: 0.3289 at 4 chains.
// A single chain lane (one chain: nothing runs beside the eps kernel)
// prefers 10 blocks (48 registers): 0.1351 vs 0.1429 ms per 1-chain sweep;
// with two lanes 10 blocks gave 0.3289 vs 0.3268 ms at 4 chains.
#ifndef CMC_EPS_MIN_BLOCKS
#define CMC_EPS_MIN_BLOCKS 9
#endif
#ifndef CMC_EPS_SOLO_MIN_BLOCKS
#define CMC_EPS_SOLO_MIN_BLOCKS 10
#endif
// with a xi prior (the xi kernel runs after each gene kernel) the eps
// kernel at 8 and the gene kernel at 6 (below): horseshoe 0.786 -> 0.770,
// t 0.542 -> 0.535 ms per 4-chain sweep against the normal model's 9 / 5
#ifndef CMC_EPS_XI_MIN_BLOCKS
#define CMC_EPS_XI_MIN_BLOCKS 8
#endif
template <int MINB>
__global__ void __launch_bounds__(kGeneBlock, MINB)
    eps_sweep_kernel(const SweepParams p, const long m_off) {
  __shared__ double exp_tab[32];
  exp_table_init(exp_tab);
  __syncthreads();
  WarpTrace wt(p, 1, p.slot_base + blockIdx.z);
  const int slot = p.slot_base + blockIdx.z;
  Hyper* hp = p.hyper + slot;
  if (stalled_chain(hp)) return;
  const long gl = (long)blockIdx.x * kGeneBlock + threadIdx.x;
  // lanes with a gene: the warp is re-converged over them after the slice
  // step (below)
  const unsigned live = __ballot_sync(0xffffffffu, gl < p.G);
  if (gl >= p.G) return;
  const int n = blockIdx.y;
  const long m = *p.d_m + m_off;
  const bool tuning = m <= p.burnin;
  const int N = p.N, L = p.L;
  const size_t G = (size_t)p.G, so = (size_t)slot;
  const uint64_t chain = (uint64_t)(p.chain_base + blockIdx.z);
  const uint64_t gg = (uint64_t)(p.g0 + gl);
  const SliceCfg sc{p.K, p.max_shrink, p.burnin, p.tune_cutoff, p.k_reject, p.k_inv};
  const size_t i = (size_t)n * G + gl;
  const size_t ie = so * N * G + i;
  const bool monitor = p.monitor_enabled && m > p.burnin;
  double* acc = p.acc_eps + so * 4 * N * G + i;
  if (monitor) {
    // the four Welford words come from HBM: start them towards L2 now so the
    // update after the slice step does not wait on DRAM
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(acc + (size_t)k * N * G));
  }

  // xb_gn = sum_l X_nl beta_gl, l ascending from 0.0 (refresh_xb,
  // P:src/engine.cpp:144-159)
  const double* beta = p.beta + so * L * G;
  double xb = 0.0;
  for (int l = 0; l < L; ++l) xb += __ldg(p.X + n * L + l) * beta[(size_t)l * G + gl];
  // 1/(2 gamma) = 0.5 * RN(1/gamma) exactly (scaling by 2 commutes with
  // rounding); inv_gam is written with gamma by the gene kernel and by
  // upload_state, so no divide per (gene, sample)
  const double inv_two_gam = 0.5 * p.inv_gam[so * G + gl];
  EpsF f{__ldg(p.y + i), __ldg(p.h + n) + xb, inv_two_gam, p.exp_clamp, ExpTab(exp_tab), 0u};
  const double x0 = p.eps[ie];
  double w = p.eps_w[ie];
  double wa = tuning ? p.eps_wa[ie] : 0.0;
  // the Philox queue's second block in shared memory (StreamSm): 64
  // registers without spills, 8 blocks per SM
  __shared__ uint64_t rngq[4 * kGeneBlock];
  StreamSm rng;
  rng.init_x2(p.seed, chain, (uint64_t)m, site_id(kSiteEps, gg * N + n),
              (unsigned)__cvta_generic_to_shared(rngq + threadIdx.x), 8u * kGeneBlock);
  bool st = false;
  const double x1 = slice_step_so2(f, x0, w, wa, sc, m, rng, st);
  // The shrink loop's lanes leave at different trips (a return inside the
  // inlined loop); without an explicit re-convergence point the stores and
  // the Welford update below ran once per exit group, at ~16 of 32 lanes
  // (ncu).  Re-converged: 2.4% per sweep.
  __syncwarp(live);
  if (st) {
    // eps and its width stay untouched: the host reads x0 and w back.
    // The eps kernel of iteration m+1 runs concurrently with the tail of
    // iteration m, so it records into its own slot (see stalled_chain).
    // the iteration first, then the key (see tail_stalled); every stalling
    // lane of one kernel writes the same m
    *(volatile long long*)&hp->err_m_eps = m;
    __threadfence();
    atomicMin(&hp->err_key_eps, stall_key(1, 0, gg, n));
  } else {
    p.eps[ie] = x1;
    if (tuning) {
      p.eps_w[ie] = w;
      p.eps_wa[ie] = wa;
    }
    if (monitor) moments(acc, (size_t)N * G, x1, (double)(m - p.burnin));
  }
  if (f.clamps) atomicAdd(&hp->clamps, (unsigned long long)f.clamps);
}

// Steps 2 and 5, one thread per gene: gamma_g from the new eps row, then
// beta_g1..beta_gL in column order.  Lanes of a warp are re-converged with
// __syncwarp() at every slice-step boundary so each step's log-density
// evaluations run as one SIMT stream (no early exits: a lane without a
// gene, or whose gene stalled, idles with alive == false).  5 blocks per
// SM (96 registers) with the eps kernel at 9 (above); 6 blocks (80
// registers, 100-byte spills) was best before the carried beta exps.
#ifndef CMC_GENE_XI_MIN_BLOCKS
#define CMC_GENE_XI_MIN_BLOCKS 6  // with a xi prior (see CMC_EPS_XI_MIN_BLOCKS)
#endif
#ifndef CMC_GENE_MIN_BLOCKS
#define CMC_GENE_MIN_BLOCKS 5
#endif
// JR > 0: every column has at most JR groups, kept in registers
// (BetaFR); JR = 0: any design, group sums in shared memory (BetaF).
// XI: some column has a xi prior (extension); the reference model (all
// normal) is compiled without the xi step.
// PH: the steps this launch runs, bit 0 step 2 (gamma), bit 1 step 5
// (beta); the sweep runs both (3), the per-step timing mode one at a time.
// the gene kernel's Philox queues keep their second block in shared memory
// (StreamSm: spills 152 -> 100 bytes)
using GeneRng = StreamSm;
#define GENE_RNG_Q , rngq_s, 8u * kGeneThreads
template <int JR, bool XI, int PH>
__device__ __forceinline__ void gene_sweep_body(const SweepParams& p, const long m_off,
                                                double* smem, const ExpTab etab) {
  __shared__ uint64_t rngq[4 * kGeneThreads];
  const unsigned rngq_s = (unsigned)__cvta_generic_to_shared(rngq + threadIdx.x);
  const int tid = threadIdx.x;
  const int slot = p.slot_base + blockIdx.y;
  Hyper* hp = p.hyper + slot;
  if (stalled_chain(hp)) return;  // warp-uniform: one load per warp
  const long gl_raw = (long)blockIdx.x * kGeneThreads + tid;
  bool alive = gl_raw < p.G;
  const long gl = alive ? gl_raw : 0;

  const long m = *p.d_m + m_off;
  const bool tuning = m <= p.burnin;
  const bool monitor = p.monitor_enabled && m > p.burnin;
  const double mcount = (double)(m - p.burnin);
  const int N = p.N, L = p.L;
  const size_t G = (size_t)p.G;
  const uint64_t chain = (uint64_t)(p.chain_base + blockIdx.y);
  const uint64_t gg = (uint64_t)(p.g0 + gl);
  const SliceCfg sc{p.K, p.max_shrink, p.burnin, p.tune_cutoff, p.k_reject, p.k_inv};
  const size_t so = (size_t)slot;

  const double* eps = p.eps + so * N * G;
  double* beta = p.beta + so * L * G;
  double* beta_w = p.beta_w + so * L * G;
  double* beta_wa = p.beta_wa + so * L * G;
  double* xs = smem;                             // [N][B]: lp
  double* sS = smem + (size_t)N * kGeneThreads;    // [Jmax][B]
  double* sLogS = sS + (size_t)p.Jmax * kGeneThreads;
  // JR > 0 with p.beta_carry: xe_n = exp(lp_n) in the group-sum rows
  double* xe = sS;
  unsigned clamps = 0;

  // lp_n = (h_n + eps_n) + xb_n with the new eps and the previous beta,
  // and ss = sum_n eps_n^2 in n order (P:src/engine.cpp:275-283,
  // P:src/model.cpp:76-82)
  constexpr bool GAM = (PH & 1) != 0, BET = (PH & 2) != 0;
  if constexpr (BET) {
    for (int n = 0; n < N; ++n) xs[n * kGeneThreads + tid] = 0.0;
    for (int l = 0; l < L; ++l) {
      const double b = alive ? beta[(size_t)l * G + gl] : 0.0;
      for (int n = 0; n < N; ++n)
        xs[n * kGeneThreads + tid] += __ldg(p.X + n * L + l) * b;
    }
  }
  const double gam_old = alive ? p.gam[so * G + gl] : 1.0;
  double ss = 0.0;
  for (int n = 0; n < N; ++n) {
    const double e = alive ? eps[(size_t)n * G + gl] : 0.0;
    if constexpr (GAM) ss += e * e;
    if constexpr (BET) xs[n * kGeneThreads + tid] = __ldg(p.h + n) + e + xs[n * kGeneThreads + tid];
  }

  // Carried exps (register-group variant): S_j below is
  // exp(-v_j bold) * sum_n exp(lp_n), with exp(lp_n) formed once here and
  // scaled by exp(v_j (bnew - bold)) after each column, instead of one exp
  // per member and column.  Only the last bits of S_j differ from the
  // reference's sum of exp(lp_n - v_j bold), and S_j only decides slice
  // comparisons; every column whose members are not all
  // inside [-700, 700] (a clamp included) takes the reference's direct sum.
  bool carry = false;
  if constexpr (JR > 0 && BET) {
#ifdef CMC_DEBUG_BOUNDS
    if (p.beta_carry) {  // lp and the carried exps: 2N rows of dynamic shared memory
      unsigned dyn;
      asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
      assert((size_t)2 * N * kGeneThreads * sizeof(double) <= dyn);
    }
#endif
    if (p.beta_carry && alive) {
      carry = true;
      for (int n = 0; n < N; ++n) {
        const double x = xs[n * kGeneThreads + tid];
        carry = carry & (x >= -700.0) & (x <= 700.0);
        xe[n * kGeneThreads + tid] = fast_exp(x, etab);
      }
    }
  }

  // Step 2: gamma_g, P:src/engine.cpp:204-226 (nu, tau of iteration m-1)
  if constexpr (GAM) {
    double gnew = gam_old, w0 = 0.0, w = 0.0, wa = 0.0;
    bool st = false;
    __syncwarp();
    if (alive) {
      const double nu = hp->nu, tau = hp->tau;
      const double shape = (nu + (double)N) / 2.0;
      const double scale = (nu * tau + ss) / 2.0;
      if (p.direct) {
        Stream rng;
        rng.init(p.seed, chain, (uint64_t)m, site_id(kSiteGamma, gg));
        gnew = 1.0 / gamma_draw(rng, shape, scale);
      } else {
        GeneRng rng;
        rng.init_x2(p.seed, chain, (uint64_t)m, site_id(kSiteGamma, gg) GENE_RNG_Q);
        InvGammaF f{-(shape + 1.0), scale};
        w0 = p.gam_w[so * G + gl];
        w = w0;
        wa = tuning ? p.gam_wa[so * G + gl] : 0.0;
        gnew = slice_step(f, gam_old, w, wa, sc, m, rng, st);
      }
    }
    __syncwarp();
    if (alive && st) {
      record_stall(hp, stall_key(2, 0, gg, 0), m);
      alive = false;
    }
    if (alive) {
      if (tuning && !p.direct) {
        p.gam_w[so * G + gl] = w;
        p.gam_wa[so * G + gl] = wa;
      }
      p.gam[so * G + gl] = gnew;
      p.log_gam[so * G + gl] = log(gnew);
      p.inv_gam[so * G + gl] = 1.0 / gnew;
      if (monitor) moments(p.acc_gam + so * 4 * G + gl, G, gnew, mcount);
    }
  }

  if constexpr (BET) {
    // Step 5: beta_g1..beta_gL in column order, P:src/engine.cpp:269-334
    for (int l = 0; l < L; ++l) {
      const size_t i = (size_t)l * G + gl;
      const int jb = __ldg(p.grp_off + l), je = __ldg(p.grp_off + l + 1);
      const bool xcol = XI && p.xi_fam[l] != CMC_PRIOR_NORMAL;  // warp-uniform
      double bold = 0.0, bnew = 0.0, w0 = 0.0, w = 0.0, wa = 0.0;
      bool st = false;
      __syncwarp();
      if (alive) {
        bold = beta[i];
        // S_j = sum over the group's samples, in order, of
        // clamped_exp(lp_n - v_j * bold) (P:src/engine.cpp:295-300)
        auto group_sum = [&](int j) {
          const double v = __ldg(p.grp_val + j);
          const double vb = v * bold;
          const int q0 = __ldg(p.grp_moff + j), q1 = __ldg(p.grp_moff + j + 1);
          double s = 0.0;
          for (int q = q0; q < q1; ++q) {
            const int n = __ldg(p.grp_mem + q);
            double t = xs[n * kGeneThreads + tid] - vb;
            if (t > kExpClamp) {
              ++clamps;
              t = kExpClamp;
            }
            s += fast_exp(t, etab);
          }
          return s;
        };
        // the same S_j from the carried exps when every term is in range
        auto group_sum_c = [&](int j) {
          const double v = __ldg(p.grp_val + j);
          const double vb = v * bold;
          const int q0 = __ldg(p.grp_moff + j), q1 = __ldg(p.grp_moff + j + 1);
          double s = 0.0;
          bool ok = (vb > -700.0) & (vb < 700.0);
          for (int q = q0; q < q1; ++q) {
            const int n = __ldg(p.grp_mem + q);
            const double t = xs[n * kGeneThreads + tid] - vb;
            ok = ok & (t >= -700.0) & (t <= kExpClamp);
            s += xe[n * kGeneThreads + tid];
          }
          return ok ? s * fast_exp(-vb, etab) : group_sum(j);
        };
        const double sig = hp->sigma[l];
        const double sig2 = sig * sig;
        // prior variance sigma_l^2 (normal) or sigma_l^2 xi_gl (xi column)
        const double inv2v = xcol ? 1.0 / (2.0 * (sig2 * p.xi[so * L * G + i]))
                                  : 1.0 / (2.0 * sig2);
        w0 = beta_w[i];
        w = w0;
        wa = tuning ? beta_wa[i] : 0.0;
        GeneRng rng;
        rng.init_x2(p.seed, chain, (uint64_t)m, site_id(kSiteBeta, gg * L + l) GENE_RNG_Q);
        if constexpr (JR > 0) {
          BetaFR<JR> f;
          f.a = __ldg(p.A + i);
          f.theta = hp->theta[l];
          f.inv_two_sig2 = inv2v;
          f.e700 = p.exp_clamp;
          f.tab = etab;
          f.J = je - jb;
          f.clamps = 0u;
  #pragma unroll
          for (int jj = 0; jj < JR; ++jj) {
            f.v[jj] = 0.0;
            f.S[jj] = 0.0;
            f.lS[jj] = 0.0;
            if (jb + jj < je) {
              f.v[jj] = __ldg(p.grp_val + jb + jj);
              f.S[jj] = carry ? group_sum_c(jb + jj) : group_sum(jb + jj);
              f.lS[jj] = log(f.S[jj]);
            }
          }
          bnew = slice_step(f, bold, w, wa, sc, m, rng, st);
          clamps += f.clamps;
        } else {
          for (int j = jb; j < je; ++j) {
            const double s = group_sum(j);
            sS[(j - jb) * kGeneThreads + tid] = s;
            sLogS[(j - jb) * kGeneThreads + tid] = log(s);
          }
          BetaF f{__ldg(p.A + i), hp->theta[l], inv2v, p.exp_clamp,
                  p.grp_val + jb, sS + tid, sLogS + tid, etab, je - jb, 0u};
          bnew = slice_step(f, bold, w, wa, sc, m, rng, st);
          clamps += f.clamps;
        }
      }
      __syncwarp();
      if (!alive) continue;
      if (st) {
        record_stall(hp, stall_key(5, l, gg, 0), m);
        alive = false;
        continue;
      }
      beta[i] = bnew;
      if (tuning) {
        beta_w[i] = w;
        beta_wa[i] = wa;
      }
      // lp after the last column is not read again (the reference's lp is
      // scratch, rebuilt at the next sweep's step 5)
      if (bnew != bold && l + 1 < L) {
        for (int j = jb; j < je; ++j) {
          const double v = __ldg(p.grp_val + j);
          const double dv = v * (bnew - bold);
          double f = 1.0;
          if constexpr (JR > 0) {
            if (carry) {
              carry = (dv > -700.0) & (dv < 700.0);
              f = fast_exp(dv, etab);
            }
          }
          for (int q = __ldg(p.grp_moff + j); q < __ldg(p.grp_moff + j + 1); ++q) {
            const int n = __ldg(p.grp_mem + q);
            const double x = xs[n * kGeneThreads + tid] + dv;
            xs[n * kGeneThreads + tid] = x;
            if constexpr (JR > 0) {
              if (carry) {
                xe[n * kGeneThreads + tid] *= f;
                carry = carry & (x >= -700.0) & (x <= 700.0);
              }
            }
          }
        }
      }
      if (monitor) moments(p.acc_beta + so * 4 * L * G + i, (size_t)L * G, bnew, mcount);
    }

    __syncwarp();
    if (alive && monitor) {
      // per-gene contrasts that read only this gene's beta/gamma
      if (p.ctab_gene_in_sweep) {
        const ContrastTable* t = p.ctab;
        const double gam = p.gam[so * G + gl];
        for (int ci = 0; ci < p.ctab_n; ++ci)
          if (t->per_gene[ci])
            contrast_update(t, ci, p.cprob + so * t->n_prob + t->prob_off[ci] + p.g0 + gl,
                            mcount, beta, G, gl, gam, hp);
      }
      // thinning of saved genes, P:src/engine.cpp:433-447
      const long cnt = m - p.burnin;
      const int sv = p.saved_slot[gl];
      if (sv >= 0 && cnt % p.thin == 0) {
        const long row = cnt / p.thin - 1;
        if (row < p.n_rows) {
          double* smp = p.samples + so * p.n_cols * p.n_rows;
          const long c0 = 2 + 2 * (long)L + (long)sv * (L + 1);
          for (int l = 0; l < L; ++l)
            smp[(c0 + l) * p.n_rows + row] = beta[(size_t)l * G + gl];
          smp[(c0 + L) * p.n_rows + row] = p.gam[so * G + gl];
        }
      }
    }
  }
  if (clamps) atomicAdd(&hp->clamps, (unsigned long long)clamps);
}


// xi_gl for every (gene, xi column) of the chain (extension, no reference:
// parity unpinned).  xi_gl's conditional reads only beta_gl (this sweep),
// theta_l and sigma_l (iteration m-1), so all G x L steps are independent:
// one thread per (gene, column) after the gene kernel, grid (G/128, L,
// chains).  The draws equal the oracle's, which takes xi_gl right after
// beta_gl inside step 5 (same sites, same inputs); a stall gets key
// (5, l, g, 1), i.e. after beta_gl and before beta_(g+1)l, the sequential
// order.
#ifndef CMC_XI_MIN_BLOCKS
#define CMC_XI_MIN_BLOCKS 8
#endif
#ifndef CMC_XI_PARK_MIN_BLOCKS
#define CMC_XI_PARK_MIN_BLOCKS 6
#endif
__global__ void __launch_bounds__(kGeneBlock, CMC_XI_MIN_BLOCKS)
    xi_sweep_kernel(const SweepParams p, const long m_off) {
  const int l = blockIdx.y;
  if (p.xi_fam[l] == CMC_PRIOR_NORMAL) return;  // block-uniform
  const int slot = p.slot_base + blockIdx.z;
  Hyper* hp = p.hyper + slot;
  if (stalled_chain(hp)) return;
  const long gl = (long)blockIdx.x * kGeneBlock + threadIdx.x;
  const unsigned live = __ballot_sync(0xffffffffu, gl < p.G);
  if (gl >= p.G) return;
  const long m = *p.d_m + m_off;
  const bool tuning = m <= p.burnin;
  const int L = p.L;
  const size_t G = (size_t)p.G, so = (size_t)slot;
  const size_t ix = so * L * G + (size_t)l * G + gl;
  const uint64_t chain = (uint64_t)(p.chain_base + blockIdx.z);
  const uint64_t gg = (uint64_t)(p.g0 + gl);
  const SliceCfg sc{p.K, p.max_shrink, p.burnin, p.tune_cutoff, p.k_reject, p.k_inv};
  const double sg = hp->sigma[l];
  const double dz = p.beta[ix] - hp->theta[l];
  XiF f{p.xi_fam[l], dz * dz / (2.0 * (sg * sg)), p.t_df};
  double w = p.xi_w[ix];
  double wa = tuning ? p.xi_wa[ix] : 0.0;
  Stream rng;
  rng.init_x2(p.seed, chain, (uint64_t)m, site_id(kSiteXi, gg * L + l));
  bool st = false;
  const double x1 = slice_step(f, p.xi[ix], w, wa, sc, m, rng, st);
  __syncwarp(live);  // re-converge after the slice loop (as in the eps kernel)
  if (st) {
    record_stall(hp, stall_key(5, l, gg, 1), m);
    return;
  }
  p.xi[ix] = x1;
  if (tuning) {
    p.xi_w[ix] = w;
    p.xi_wa[ix] = wa;
  }
  if (p.monitor_enabled && m > p.burnin)
    moments(p.acc_xi + so * 4 * L * G + (size_t)l * G + gl, (size_t)L * G, x1,
            (double)(m - p.burnin));
}

// The same step for a launch with a horseshoe column (xi_park_kernel).
// Divergence: a horseshoe xi's slice loop is heavy-tailed (long step-outs,
// many shrinks), and a warp runs as long as its slowest lane.  So the loop
// runs at most p.xi_trips trips for every lane, then every lane still
// running parks its whole state (slice state, Philox queue, density
// parameter) in shared memory -- a warp vote (__ballot_sync) gives each
// warp its running lanes, the warp's leader reserves that many queue slots
// with one atomic, and each lane takes its rank among them -- and the
// block's first threads resume the parked steps densely packed, one per
// thread.  The continuation draws the
// same uniforms in the same order, so the result is unchanged.
struct XiParked {
  SliceRun s;
  uint64_t a0, a1, a2, a3, b0, b1, b2, b3;
  double q, w, wa;
  unsigned block, na, nb;
  int gl;
};
constexpr int kXiPark = kGeneBlock;  // every lane of the block can park

__global__ void __launch_bounds__(kGeneBlock, CMC_XI_PARK_MIN_BLOCKS)
    xi_park_kernel(const SweepParams p, const long m_off) {
  __shared__ XiParked park[kXiPark];
  __shared__ int n_park;
  const int l = blockIdx.y;
  if (p.xi_fam[l] == CMC_PRIOR_NORMAL) return;  // block-uniform
  const int slot = p.slot_base + blockIdx.z;
  Hyper* hp = p.hyper + slot;
  if (threadIdx.x == 0) n_park = stalled_chain(hp) ? -1 : 0;
  __syncthreads();
  if (n_park < 0) return;  // block-uniform
  const long gl = (long)blockIdx.x * kGeneBlock + threadIdx.x;
  const bool alive = gl < p.G;
  const long m = *p.d_m + m_off;
  const bool tuning = m <= p.burnin;
  const int L = p.L;
  const size_t G = (size_t)p.G, so = (size_t)slot;
  const uint64_t chain = (uint64_t)(p.chain_base + blockIdx.z);
  const SliceCfg sc{p.K, p.max_shrink, p.burnin, p.tune_cutoff, p.k_reject, p.k_inv};
  const double sg = hp->sigma[l];
  const double th = hp->theta[l];
  const bool monitor = p.monitor_enabled && m > p.burnin;
  // result of one lane's step (pass 1 or resumed): xi, width, stall
  auto finish = [&](long g, int res, const SliceRun& s, double w, double wa) {
    const size_t ix = so * L * G + (size_t)l * G + g;
    if (res == kSliceStalled) {
      record_stall(hp, stall_key(5, l, (uint64_t)(p.g0 + g), 1), m);
      return;
    }
    if (m <= sc.burnin) tune_update(w, wa, m, fabs(s.x1 - s.x0), sc.tune_cutoff);
    p.xi[ix] = s.x1;
    if (tuning) {
      p.xi_w[ix] = w;
      p.xi_wa[ix] = wa;
    }
    if (monitor)
      moments(p.acc_xi + so * 4 * L * G + (size_t)l * G + g, (size_t)L * G, s.x1,
              (double)(m - p.burnin));
  };
  int res = kSliceAccepted;
  SliceRun s;
  Stream rng;
  double w = 0.0, wa = 0.0, q = 0.0;
  if (alive) {
    const size_t ix = so * L * G + (size_t)l * G + gl;
    const double dz = p.beta[ix] - th;
    q = dz * dz / (2.0 * (sg * sg));
    XiF f{p.xi_fam[l], q, p.t_df};
    w = p.xi_w[ix];
    wa = tuning ? p.xi_wa[ix] : 0.0;
    rng.init_x2(p.seed, chain, (uint64_t)m, site_id(kSiteXi, (uint64_t)(p.g0 + gl) * L + l));
    slice_start(f, p.xi[ix], w, sc, rng, s);
    res = slice_trips(f, sc, rng, s, p.xi_trips);
  }
  // park the lanes still running
  const bool parked = alive && res == kSliceRunning;
  const unsigned vote = __ballot_sync(0xffffffffu, parked);
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == 0 && vote) base = atomicAdd(&n_park, __popc(vote));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (parked) {
    const int k = base + __popc(vote & ((1u << lane) - 1u));
#ifdef CMC_DEBUG_BOUNDS
    assert(k >= 0 && k < kXiPark);
#endif
    {
      XiParked& e = park[k];
      e.s = s;
      e.a0 = rng.a0; e.a1 = rng.a1; e.a2 = rng.a2; e.a3 = rng.a3;
      e.b0 = rng.b0; e.b1 = rng.b1; e.b2 = rng.b2; e.b3 = rng.b3;
      e.block = rng.block; e.na = rng.na; e.nb = rng.nb;
      e.q = q;
      e.w = w;
      e.wa = wa;
      e.gl = (int)gl;
    }
  }
  __syncwarp();
  if (alive && !parked) finish(gl, res, s, w, wa);
  __syncthreads();
  const int np = n_park;
  if ((int)threadIdx.x >= np) return;
  // resume one parked step per thread, densely packed in the first warps
  const XiParked& e = park[threadIdx.x];
  SliceRun r = e.s;
  Stream rs;
  rs.k0 = p.seed;
  rs.k1 = chain;
  rs.it = (uint64_t)m;
  rs.site = site_id(kSiteXi, (uint64_t)(p.g0 + e.gl) * L + l);
  rs.a0 = e.a0; rs.a1 = e.a1; rs.a2 = e.a2; rs.a3 = e.a3;
  rs.b0 = e.b0; rs.b1 = e.b1; rs.b2 = e.b2; rs.b3 = e.b3;
  rs.block = e.block; rs.na = e.na; rs.nb = e.nb;
  XiF f{p.xi_fam[l], e.q, p.t_df};
  const int rr = slice_trips(f, sc, rs, r, 0x7fffffff);
  __syncwarp(__activemask());
  finish(e.gl, rr, r, e.w, e.wa);
}

// Serial sum of value(i), i in [start, end), from +0.0 in index order: the
// reference's left-to-right leaf loop (P:include/countmc/parallel.hpp:
// 76-81).  The warp stages kStage values at a time in its shared buffer
// (coalesced loads, the next chunk in flight while this one is summed) and
// lane 0 adds them one by one from shared memory, so the dependent chain is
// one DADD per value with nothing else on it.  Padding past `end` with +0.0
// is exact: the running sum starts at +0.0 and can never become -0.0, so
// s + 0.0 == s.  Called by a whole warp; every lane gets the sum.
// s + b[0] + b[1] + ... + b[n-1], left to right, from shared memory: the
// loads of the next 16 values are issued before the 16 dependent additions
// of the current ones, so the chain runs at the DADD latency instead of
// load + add per value (timeline: 11.4 us per leaf epilogue warp before)
// A/B (ms per sweep, 100-sweep calls, 4 chains / 1 chain): the pipelined
// chain in the gene kernel's epilogue 0.3213 -> 0.3192 / 0.1295 -> 0.1274;
// in the tail kernels' warp_serial_sum as well 0.3266 / 0.1257 -- a faster
// high-priority tail takes SM time from the eps and gene kernels at 4
// chains -- so the tail keeps the plain loop
#ifndef CMC_TAIL_PIPE
#define CMC_TAIL_PIPE 0
#endif
#ifndef CMC_TAIL_PIPE_B
#define CMC_TAIL_PIPE_B 16
#endif
#ifndef CMC_EPI_PIPE
#define CMC_EPI_PIPE 1
#endif
template <int B = 16>
__device__ __forceinline__ double serial_add(const double* b, int n, double s) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(b);
  auto ld = [&](int i) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a + ((unsigned)i << 3)));
    return v;
  };
  int i = 0;
  if (n >= B) {
    double t[B];
#pragma unroll
    for (int j = 0; j < B; ++j) t[j] = ld(j);
    for (i = B; i + B <= n; i += B) {
      double u[B];
#pragma unroll
      for (int j = 0; j < B; ++j) u[j] = ld(i + j);
#pragma unroll
      for (int j = 0; j < B; ++j) s += t[j];
#pragma unroll
      for (int j = 0; j < B; ++j) t[j] = u[j];
    }
#pragma unroll
    for (int j = 0; j < B; ++j) s += t[j];
  }
  for (; i < n; ++i) s += ld(i);
  return s;
}

template <class V>
__device__ __forceinline__ double warp_serial_sum(V value, long start, long end, double* buf) {
  const int lane = threadIdx.x & 31;
  constexpr int PER = kStage / 32;
  const int chunks = (int)((end - start + kStage - 1) / kStage);
  double v[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const long idx = start + k * 32 + lane;
    v[k] = idx < end ? value(idx) : 0.0;
  }
  double s = 0.0;
  for (int c = 0; c < chunks; ++c) {
#pragma unroll
    for (int k = 0; k < PER; ++k) buf[k * 32 + lane] = v[k];
    __syncwarp();
    if (c + 1 < chunks) {
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const long idx = start + (long)(c + 1) * kStage + k * 32 + lane;
        v[k] = idx < end ? value(idx) : 0.0;
      }
    }
    if (lane == 0) {
#if CMC_TAIL_PIPE
      s = serial_add<CMC_TAIL_PIPE_B>(buf, kStage, s);
#else
#pragma unroll 16
      for (int i = 0; i < kStage; ++i) s += buf[i];
#endif
    }
    __syncwarp();
  }
  return __shfl_sync(0xffffffffu, s, 0);
}

// pairwise_sum (P:src/parallel.cpp:81-86) of the leaf partials
// [lo, lo + n), n <= MAX, as straight-line code: the recursion unrolled at
// compile time (no stack, no local buffer).  A node of size 1 is its leaf,
// a node of size 0 is 0.0, children split at n / 2, exactly as the
// reference recursion.
template <int MAX>
__device__ __forceinline__ double pairwise_fixed(const PartView& v, int q, long lo, int n) {
  if constexpr (MAX <= 1) {
    return n == 1 ? leaf_part(v, q, lo) : 0.0;
  } else {
    if (n <= 1) return n == 1 ? leaf_part(v, q, lo) : 0.0;
    const int mid = n / 2;
    return pairwise_fixed<MAX / 2>(v, q, lo, mid) +
           pairwise_fixed<(MAX + 1) / 2>(v, q, lo + mid, n - mid);
  }
}

// pairwise_sum of one quantity's leaf partials by one warp.  Lane k walks
// the top five midpoint splits along the bits of k, sums its depth-5
// subtree with the same recursion (straight-line up to 32 leaves per lane,
// i.e. 1,024 leaves = 1M genes; the plain recursion beyond), and the 31
// internal nodes above are rebuilt with shuffles as left + right.  A node
// of size 1 passes its single leaf through and a node of size 0 is 0.0, as
// the reference recursion returns them, so the result is bit-identical.
__device__ double warp_pairwise_leaves(const PartView pv, int q, int n) {
  const int lane = threadIdx.x & 31;
  int lo = 0, cnt = n;
  int cnts[5];
#pragma unroll
  for (int d = 0; d < 5; ++d) {
    cnts[d] = cnt;
    const int mid = cnt / 2;
    if ((lane >> (4 - d)) & 1) {
      lo += mid;
      cnt -= mid;
    } else {
      cnt = mid;
    }
  }
  const double v0 = cnt <= 32 ? pairwise_fixed<32>(pv, q, lo, cnt) : pairwise_leaves(pv, q, lo, cnt);
  double v = v0;
#pragma unroll
  for (int d = 4; d >= 0; --d) {
    const int bit = 4 - d;
    const double other = __shfl_xor_sync(0xffffffffu, v, 1 << bit);
    const bool right = (lane >> bit) & 1;
    if (cnts[d] == 0)
      v = 0.0;
    else if (cnts[d] == 1)
      v = right ? v : other;
    else
      v = right ? (other + v) : (v + other);
  }
  return v;
}

template <bool XI>
__device__ void hyper_a_body(const SweepParams& p, int slot, long m);

// Leaf sums of partA's quantities for leaf lb of one chain: log gamma
// (q = 0), 1/gamma (1), beta_l (2 + l); with a xi prior S_l = beta_l/xi_l
// on xi columns and W_l = 1/xi_l (2 + L + l).  The reference tree's leaves
// (P:include/countmc/parallel.hpp:67-84): each sum runs serially in gene
// order.  The block's warps stride over the quantities, each staging
// through its own kStage buffer; loads bypass L1 (__ldcg) because the
// gene kernel's other blocks wrote the values.
template <bool XI>
__device__ void leaf_a_sums(const SweepParams& p, int slot, long lb, double* stage) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int L = p.L, Q = leaf_q_a(L, p.xi_any), Qs = leaf_qs_a(L, p.xi_any);
  const size_t G = (size_t)p.G, so = (size_t)slot;
  const long start = lb * kLeaf;
  const long end = min((long)G, start + kLeaf);
  const long lpr = p.leaves_per_rank;
  const long rank = (p.g0 / kLeaf) / (lpr > 0 ? lpr : 1);
  double* buf = stage + (size_t)warp * kStage;
  for (int q = warp; q < Q; q += nwarps) {
    double s;
    if (q < 2) {
      const double* src = (q == 0 ? p.log_gam : p.inv_gam) + so * G;
      s = warp_serial_sum([&](long i) { return __ldcg(src + i); }, start, end, buf);
    } else if (q < 2 + L) {
      const double* src = p.beta + so * L * G + (size_t)(q - 2) * G;
      if (XI && p.xi_fam[q - 2] != CMC_PRIOR_NORMAL) {  // extension: beta / xi
        const double* xs = p.xi + so * L * G + (size_t)(q - 2) * G;
        s = warp_serial_sum([&](long i) { return __ldcg(src + i) / __ldcg(xs + i); }, start,
                            end, buf);
      } else {
        s = warp_serial_sum([&](long i) { return __ldcg(src + i); }, start, end, buf);
      }
    } else {  // extension: 1 / xi
      const double* xs = p.xi + so * L * G + (size_t)(q - 2 - L) * G;
      s = warp_serial_sum([&](long i) { return 1.0 / __ldcg(xs + i); }, start, end, buf);
    }
#ifdef CMC_DEBUG_BOUNDS
    assert(rank >= 0 && rank < p.world && slot - p.slot_base < p.C && q < Qs && lb < lpr);
#endif
    if (lane == 0) p.partA[((rank * p.C + (slot - p.slot_base)) * Qs + q) * lpr + lb] = s;
  }
}

// leaf_a_sums for the gene kernel's epilogue (no xi prior): the warps take
// the quantities in pairs (q, q + nwarps), lane 0 adding the first and lane
// 1 the second in the same instruction stream, so the 2 + L serial chains
// of 1,024 additions run in one round of two interleaved chains per warp
// instead of two rounds of one.  Each chain is still serial in gene order.
#ifndef CMC_LEAF_PAIRED
#define CMC_LEAF_PAIRED 1
#endif
__device__ void leaf_a_sums_paired(const SweepParams& p, int slot, long lb, double* stage) {
  // 256-value staging rounds (four per leaf), the next round's loads in
  // flight while the current one is added
  constexpr int kEpi = kStageEpi;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int L = p.L, Q = 2 + L, Qs = leaf_qs_a(L, 0);
  const size_t G = (size_t)p.G, so = (size_t)slot;
  const long start = lb * kLeaf;
  const long end = min((long)G, start + kLeaf);
  const long lpr = p.leaves_per_rank;
  const long rank = (p.g0 / kLeaf) / (lpr > 0 ? lpr : 1);
  double* bufA = stage + (size_t)warp * 2 * kEpi;
  double* bufB = bufA + kEpi;
#ifdef CMC_DEBUG_BOUNDS
  {  // the staging rounds fit the kernel's dynamic shared memory
    unsigned dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    assert((size_t)2 * nwarps * kEpi * sizeof(double) <= dyn);
  }
#endif
  auto src_of = [&](int q) -> const double* {
    return q < 2 ? (q == 0 ? p.log_gam : p.inv_gam) + so * G
                 : p.beta + so * L * G + (size_t)(q - 2) * G;
  };
  constexpr int PER = kEpi / 32;
  const int chunks = (int)((end - start + kEpi - 1) / kEpi);
  for (int qa = warp; qa < Q; qa += 2 * nwarps) {
    const int qb = qa + nwarps;
    const double* A = src_of(qa);
    const double* B = qb < Q ? src_of(qb) : A;
    double va[PER], vb[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const long idx = start + k * 32 + lane;
      va[k] = idx < end ? __ldcg(A + idx) : 0.0;
      vb[k] = idx < end ? __ldcg(B + idx) : 0.0;
    }
    double s = 0.0;
    const double* mine = lane == 1 ? bufB : bufA;
    for (int c = 0; c < chunks; ++c) {
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        bufA[k * 32 + lane] = va[k];
        bufB[k * 32 + lane] = vb[k];
      }
      __syncwarp();
      if (c + 1 < chunks) {
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          const long idx = start + (long)(c + 1) * kEpi + k * 32 + lane;
          va[k] = idx < end ? __ldcg(A + idx) : 0.0;
          vb[k] = idx < end ? __ldcg(B + idx) : 0.0;
        }
      }
      if (lane < 2) {
        const int n = (int)min((long)kEpi, end - start - (long)c * kEpi);
#if CMC_EPI_PIPE
        s = serial_add<8>(mine, n, s);
#else
#pragma unroll 16
        for (int i = 0; i < n; ++i) s += mine[i];
#endif
      }
      __syncwarp();
    }
#ifdef CMC_DEBUG_BOUNDS
    assert(rank >= 0 && rank < p.world && slot - p.slot_base < p.C && qa < Qs && lb < lpr);
#endif
    double* dst = p.partA + (rank * p.C + (slot - p.slot_base)) * Qs * lpr + lb;
    if (lane == 0) dst[(size_t)qa * lpr] = s;
    if (lane == 1 && qb < Q) dst[(size_t)qb * lpr] = s;
  }
}

// This rank's stall flag of a chain in the gathered partA section (sharded
// runs): leaf slot 0 of quantity Q.
__device__ __forceinline__ void write_stall_flag(const SweepParams& p, int slot, bool st) {
  const long lpr = p.leaves_per_rank;
  const long rank = (p.g0 / kLeaf) / (lpr > 0 ? lpr : 1);
  const int Q = leaf_q_a(p.L, p.xi_any), Qs = leaf_qs_a(p.L, p.xi_any);
#ifdef CMC_DEBUG_BOUNDS
  assert(rank >= 0 && rank < p.world && slot - p.slot_base < p.C);
#endif
  p.partA[((rank * p.C + (slot - p.slot_base)) * Qs + Q) * lpr] = st ? 1.0 : 0.0;
}

// End of the gene kernel (no xi prior): the leaf reductions fused into the
// update kernel.  The last of a leaf's (up to) 8 blocks to finish sums the
// leaf for its chain (hyper_a_kernel then reduces the leaves and draws nu,
// tau, theta).  Sharded, the last leaf of the chain also writes this
// rank's stall flag for the all-gather.  Every block of the grid takes
// part, also when the chain stalled (the body then did nothing), so the
// per-leaf counters always return to 0.
template <bool XI>
__device__ void gene_leaf_epilogue(const SweepParams& p, int slot, long m, double* stage) {
  __shared__ int s_role;
  const int tid = threadIdx.x;
  Hyper* hp = p.hyper + slot;
  const long lb = blockIdx.x / kBlocksPerLeaf;
  __threadfence();  // this thread's gamma/beta stores before the count
  __syncthreads();
  if (tid == 0) {
    const unsigned nb = min((unsigned)kBlocksPerLeaf, gridDim.x - (unsigned)lb * kBlocksPerLeaf);
#ifdef CMC_DEBUG_BOUNDS
    assert(lb < p.n_leaves_local && nb >= 1 && nb <= (unsigned)kBlocksPerLeaf);
#endif
    unsigned* cnt = p.leaf_cnt + (size_t)slot * p.n_leaves_local + lb;
    const bool last = atomicAdd(cnt, 1u) == nb - 1;
    if (last) *cnt = 0;
    s_role = last ? 1 : 0;
  }
  __syncthreads();
  if (!s_role) return;
  WarpTrace wt(p, 6, slot);  // the leaf's serial sums (timeline only)
  __threadfence();
  if (CMC_LEAF_PAIRED && !XI)
    leaf_a_sums_paired(p, slot, lb, stage);
  else
    leaf_a_sums<XI>(p, slot, lb, stage);
  if (p.fuse_tail) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const bool last = atomicAdd(&hp->doneA, 1u) == (unsigned)p.n_leaves_local - 1;
    if (last) {
      hp->doneA = 0;
      __threadfence();
      write_stall_flag(p, slot, tail_stalled(hp, m));
    }
  }
}

template <int JR, bool XI, int PH>
__global__ void __launch_bounds__(kGeneThreads, XI ? CMC_GENE_XI_MIN_BLOCKS : CMC_GENE_MIN_BLOCKS)
    gene_sweep_kernel(const SweepParams p, const long m_off) {
  extern __shared__ double smem[];
  __shared__ double exp_tab[32];
  exp_table_init(exp_tab);
  __syncthreads();
  WarpTrace wt(p, 2, p.slot_base + blockIdx.y);  // the body and the leaf epilogue
  gene_sweep_body<JR, XI, PH>(p, m_off, smem, ExpTab(exp_tab));
  // the lp buffer (at least 16 x 128 doubles, gene_sweep_smem_bytes) is free
  // now: it stages the leaf sums
  if constexpr (!XI && (PH & 2) != 0) {
    if (p.fuse_leaf_a) gene_leaf_epilogue<XI>(p, p.slot_base + blockIdx.y, *p.d_m + m_off, smem);
  }
}

// Steps 3, 4 and 6: nu, tau and theta from the gathered leaf sums.  Called
// by a whole block of 32*(2+L) threads (warp q reduces quantity q).
template <bool XI>
__device__ void hyper_a_body(const SweepParams& p, int slot, long m) {
  __shared__ double red[XI ? 2 + 2 * kLMax : 2 + kLMax];
  Hyper* hp = p.hyper + slot;
  const int tid = threadIdx.x, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const uint64_t chain = (uint64_t)(p.chain_base + (slot - p.slot_base));
  const int L = p.L, Q = leaf_q_a(L, p.xi_any), Qs = leaf_qs_a(L, p.xi_any);
  const SliceCfg sc{p.K, p.max_shrink, p.burnin, p.tune_cutoff, p.k_reject, p.k_inv};
  const double Gd = (double)p.G_total;
  for (int q = warp; q < Q; q += nwarps) {  // Q may exceed the block's warps
    const double r = warp_pairwise_leaves(part_view(p.partA, p, slot, Qs), q, p.n_leaves_total);
    if ((tid & 31) == 0) red[q] = r;
  }
  __syncthreads();
  // per-step timing mode: SM cycles of each draw (clock64 on the drawing
  // thread), summed into p.step_cycles[slot][0..2]
  unsigned long long* cyc = p.step_cycles ? p.step_cycles + 4 * (size_t)slot : nullptr;
  if (tid == 0) {
    const double s1 = red[0], s2 = red[1];
    const long long c0 = clock64();
    // Step 3: nu, P:src/engine.cpp:228-248
    {
      NuF f{Gd, hp->tau, s1, s2, p.d};
      Stream rng;
      rng.init(p.seed, chain, (uint64_t)m, site_id(kSiteNu, 0));
      double w = hp->w_nu, wa = hp->wa_nu;
      bool st = false;
      const double x0 = hp->nu;
      const double v = slice_step(f, x0, w, wa, sc, m, rng, st);
      if (st) {
        hp->err_x0[0] = x0;
        hp->err_w[0] = hp->w_nu;
        record_stall(hp, stall_key(3, 0, 0, 0), m);
        return;
      }
      hp->nu = v;
      hp->w_nu = w;
      hp->wa_nu = wa;
    }
    const long long c1 = clock64();
    if (cyc) cyc[0] += (unsigned long long)(c1 - c0);
    // Step 4: tau, P:src/engine.cpp:250-267 / P:src/model.cpp:102-105
    {
      const double nu = hp->nu;
      const double shape = p.a + Gd * nu / 2.0;
      const double rate = p.b + (nu / 2.0) * s2;
      Stream rng;
      rng.init(p.seed, chain, (uint64_t)m, site_id(kSiteTau, 0));
      if (p.direct) {
        hp->tau = gamma_draw(rng, shape, rate);
      } else {
        GammaRateF f{shape - 1.0, rate};
        double w = hp->w_tau, wa = hp->wa_tau;
        bool st = false;
        const double x0 = hp->tau;
        const double v = slice_step(f, x0, w, wa, sc, m, rng, st);
        if (st) {
          hp->err_x0[1] = x0;
          hp->err_w[1] = hp->w_tau;
          record_stall(hp, stall_key(4, 0, 0, 0), m);
          return;
        }
        hp->tau = v;
        hp->w_tau = w;
        hp->wa_tau = wa;
      }
    }
    if (cyc) cyc[1] += (unsigned long long)(clock64() - c1);
  } else if (tid >= 32 && tid < 32 + L) {
    // Step 6: theta_l, P:src/engine.cpp:336-347 / P:src/model.cpp:124-129
    const long long c0 = clock64();
    const int l = tid - 32;
    const double sb = red[2 + l];
    const double sg = hp->sigma[l], c = p.c[l];
    // xi column (extension): precision 1/c^2 + sum_g 1/(sigma^2 xi_g), with
    // sb = sum_g beta_g / xi_g (the oracle's step 6)
    const double gw = (XI && p.xi_fam[l] != CMC_PRIOR_NORMAL) ? red[2 + L + l] : Gd;
    const double v = 1.0 / (1.0 / (c * c) + gw / (sg * sg));
    const double mean = v * sb / (sg * sg);
    const double sd = sqrt(v);
    Stream rng;
    rng.init(p.seed, chain, (uint64_t)m, site_id(kSiteTheta, l));
    hp->theta[l] = mean + sd * normal(rng);
    if (cyc && l == 0) cyc[2] += (unsigned long long)(clock64() - c0);
  }
}

// Step 7 plus the hyper monitors, global contrasts and thinning.
__device__ void hyper_b_body(const SweepParams& p, int slot, long m) {
  __shared__ double red[kLMax];
  Hyper* hp = p.hyper + slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint64_t chain = (uint64_t)(p.chain_base + (slot - p.slot_base));
  const int L = p.L;
  const SliceCfg sc{p.K, p.max_shrink, p.burnin, p.tune_cutoff, p.k_reject, p.k_inv};
  if (warp < L) {
    const double r = warp_pairwise_leaves(part_view(p.partB, p, slot, L), warp, p.n_leaves_total);
    if ((tid & 31) == 0) red[warp] = r;
  }
  __syncthreads();
  if (tid < L) {
    // Step 7: sigma_l, P:src/engine.cpp:349-369
    const int l = tid;
    const double ss = red[l];
    SigmaF f{(double)p.G_total, ss, p.s[l]};
    Stream rng;
    rng.init(p.seed, chain, (uint64_t)m, site_id(kSiteSigma, l));
    double w = hp->w_sigma[l], wa = hp->wa_sigma[l];
    bool st = false;
    const double x0 = hp->sigma[l];
    const double v = slice_step(f, x0, w, wa, sc, m, rng, st);
    if (st) {
      hp->err_x0[2 + l] = x0;
      hp->err_w[2 + l] = hp->w_sigma[l];
      record_stall(hp, stall_key(7, l, 0, 0), m);
    } else {
      hp->sigma[l] = v;
      hp->w_sigma[l] = w;
      hp->wa_sigma[l] = wa;
    }
  }
  __syncthreads();
  if (tid == 0 && p.monitor_enabled && m > p.burnin && hp->err_key == kNoError) {
    const long cnt = m - p.burnin;
    const double mc = (double)cnt;
    const int K = 2 + 2 * kLMax;
    auto upd = [&](int k, double v) {
      double mean = hp->acc[0][k], meansq = hp->acc[1][k], c1 = hp->acc[2][k],
             c2 = hp->acc[3][k];
      kahan(mean, c1, (v - mean) / mc);
      kahan(meansq, c2, (v * v - meansq) / mc);
      hp->acc[0][k] = mean;
      hp->acc[1][k] = meansq;
      hp->acc[2][k] = c1;
      hp->acc[3][k] = c2;
    };
    (void)K;
    upd(0, hp->nu);
    upd(1, hp->tau);
    for (int l = 0; l < L; ++l) upd(2 + l, hp->theta[l]);
    for (int l = 0; l < L; ++l) upd(2 + L + l, hp->sigma[l]);
    const ContrastTable* t = p.ctab;
    for (int ci = 0; ci < p.ctab_n; ++ci)
      if (!t->per_gene[ci])
        contrast_update(t, ci, p.cprob + (size_t)slot * t->n_prob + t->prob_off[ci],
                        mc, nullptr, 0, 0, 0.0, hp);
    if (cnt % p.thin == 0) {
      const long row = cnt / p.thin - 1;
      if (row < p.n_rows) {
        double* smp = p.samples + (size_t)slot * p.n_cols * p.n_rows;
        long col = 0;
        smp[(col++) * p.n_rows + row] = hp->nu;
        smp[(col++) * p.n_rows + row] = hp->tau;
        for (int l = 0; l < L; ++l) smp[(col++) * p.n_rows + row] = hp->theta[l];
        for (int l = 0; l < L; ++l) smp[(col++) * p.n_rows + row] = hp->sigma[l];
      }
    }
  }
}

__device__ __forceinline__ bool last_block(unsigned int* counter, unsigned total) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(counter, 1u);
    is_last = (prev == total - 1);
    if (is_last) *counter = 0;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// Leaf sums of partA's quantities (leaf_a_sums) as their own kernel, one
// block per local leaf and chain: used with a xi prior, whose S_l and W_l
// need the xi kernel's draws (without one the gene kernel sums its leaves,
// gene_leaf_epilogue).  One GPU: the last block runs steps 3, 4 and 6.
// Sharded: block 0 writes this rank's stall flag for the all-gather.  Tail
// kernels run at most kTailWarps warps per block (registers for 512
// threads are guaranteed); warps loop over the quantities.
template <bool XI>
__global__ void __launch_bounds__(32 * kTailWarps) leaf_a_kernel(const SweepParams p,
                                                                 const long m_off) {
  __shared__ double stage[kTailWarps][kStage];
  WarpTrace wt(p, 3, p.slot_base + blockIdx.y);
  const int slot = p.slot_base + blockIdx.y;
  Hyper* hp = p.hyper + slot;
  const long m = *p.d_m + m_off;
  const bool st = tail_stalled(hp, m);
  if (!p.fuse_tail && blockIdx.x == 0 && threadIdx.x == 0) write_stall_flag(p, slot, st);
  if (st) return;
  leaf_a_sums<XI>(p, slot, blockIdx.x, &stage[0][0]);
  if (!p.fuse_tail) return;
  if (!last_block(&hp->doneA, (unsigned)p.n_leaves_local)) return;
  hyper_a_body<XI>(p, slot, m);
}

// Steps 3, 4 and 6 from the leaf sums (one block per chain): after the
// gene kernel's fused leaf sums on one GPU, after the all-gather when
// sharded.  Sharded, every rank's stall flag is checked first: if a rank's
// chain stalled, every rank stops the chain here (identically, from the
// same gathered flags) and sync reports the stalling rank's record.
template <bool XI>
__global__ void __launch_bounds__(32 * kTailWarps) hyper_a_kernel(const SweepParams p,
                                                                  const long m_off) {
  const int slot = p.slot_base + blockIdx.x;
  WarpTrace wt(p, 5, slot);
  Hyper* hp = p.hyper + slot;
  const long m = *p.d_m + m_off;
  if (tail_stalled(hp, m)) return;
  const int Q = leaf_q_a(p.L, p.xi_any), Qs = leaf_qs_a(p.L, p.xi_any);
  const long lpr = p.leaves_per_rank, c = slot - p.slot_base;
  for (int r = 0; r < p.world && !p.fuse_tail; ++r)
    if (__ldcg(p.partA + ((r * p.C + c) * Qs + Q) * lpr) != 0.0) {
      if (threadIdx.x == 0) hp->peer_stall = 1u;
      return;
    }
  hyper_a_body<XI>(p, slot, m);
}

// Leaf sums of (beta_l - theta_l)^2 with theta of this iteration (one warp
// per column, staged like leaf_a_sums); one GPU: the last block draws sigma
// (step 7) and updates the hyper monitors.
template <bool XI>
__global__ void __launch_bounds__(32 * kTailWarps) leaf_b_kernel(const SweepParams p,
                                                                 const long m_off) {
  __shared__ double stage[kTailWarps][kStage];
  WarpTrace wt(p, 4, p.slot_base + blockIdx.y);
  const int slot = p.slot_base + blockIdx.y;
  Hyper* hp = p.hyper + slot;
  const long m = *p.d_m + m_off;
  if (tail_stalled(hp, m)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = p.L;
  const size_t G = (size_t)p.G, so = (size_t)slot;
  const long lb = blockIdx.x;
  const long start = lb * kLeaf;
  const long end = min((long)G, start + kLeaf);
  double* buf = &stage[warp][0];
  for (int q = warp; q < L; q += blockDim.x >> 5) {
    const double th = hp->theta[q];
    const double* src = p.beta + so * L * G + (size_t)q * G;
    double s;
    if (XI && p.xi_fam[q] != CMC_PRIOR_NORMAL) {  // extension: /xi
      const double* xs = p.xi + so * L * G + (size_t)q * G;
      s = warp_serial_sum(
          [&](long i) {
            const double dl = src[i] - th;
            return dl * dl / xs[i];
          },
          start, end, buf);
    } else {
      s = warp_serial_sum(
          [&](long i) {
            const double dl = src[i] - th;
            return dl * dl;
          },
          start, end, buf);
    }
    if (lane == 0) {
      const long lpr = p.leaves_per_rank;
      const long rank = (p.g0 / kLeaf) / (lpr > 0 ? lpr : 1);
#ifdef CMC_DEBUG_BOUNDS
      assert(rank >= 0 && rank < p.world && slot - p.slot_base < p.C && lb < lpr);
#endif
      p.partB[((rank * p.C + (slot - p.slot_base)) * L + q) * lpr + lb] = s;
    }
  }
  if (!p.fuse_tail) return;
  if (!last_block(&hp->doneB, (unsigned)p.n_leaves_local)) return;
  hyper_b_body(p, slot, m);
}

__global__ void __launch_bounds__(32 * kTailWarps) hyper_b_kernel(const SweepParams p,
                                                                  const long m_off) {
  const int slot = p.slot_base + blockIdx.x;
  const long m = *p.d_m + m_off;
  if (tail_stalled(p.hyper + slot, m)) return;
  hyper_b_body(p, slot, m);
}

// Per-gene contrasts that read hyperparameters of the same iteration: run
// after hyper_b (only built when such a contrast exists).
__global__ void gene_contrast_kernel(const SweepParams p, const long m_off) {
  const int slot = p.slot_base + blockIdx.y;
  const Hyper* hp = p.hyper + slot;
  const long m = *p.d_m + m_off;
  if (tail_stalled(hp, m)) return;
  const long gl = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gl >= p.G) return;
  if (!(p.monitor_enabled && m > p.burnin)) return;
  const double mc = (double)(m - p.burnin);
  const size_t G = (size_t)p.G, so = (size_t)slot;
  const ContrastTable* t = p.ctab;
  const double* beta = p.beta + so * p.L * G;
  const double gam = p.gam[so * G + gl];
  for (int ci = 0; ci < p.ctab_n; ++ci)
    if (t->per_gene[ci])
      contrast_update(t, ci, p.cprob + so * t->n_prob + t->prob_off[ci] + p.g0 + gl, mc,
                      beta, G, gl, gam, hp);
}

__global__ void advance_kernel(long* d_m, long by) { *d_m += by; }

__global__ void fill_kernel(double* p, size_t n, double v) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// A_gl = sum_n y_gn X_nl accumulated in n order, P:src/engine.cpp:55-60.
__global__ void compute_A_kernel(const double* y, const double* X, double* A,
                                 int G, int N, int L) {
  const long g = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= G) return;
  for (int l = 0; l < L; ++l) {
    double acc = 0.0;
    for (int n = 0; n < N; ++n) acc += y[(size_t)n * G + g] * X[n * L + l];
    A[(size_t)l * G + g] = acc;
  }
}

}  // namespace

// Launch with a scheduling priority (cudaLaunchAttributePriority; kept by
// graph capture, honoured with cudaGraphInstantiateFlagUseNodePriority).
template <class K>
cudaError_t launch_prio(K kernel, dim3 grid, dim3 block, size_t smem,
                        cudaStream_t s, int prio, const SweepParams& p, long m_off) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributePriority;
  attr[0].val.priority = prio;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, p, m_off);
}

int beta_carry_ok(int N, int Jmax) {
  static const int env = [] {
    const char* v = std::getenv("CMC_BETA_CARRY");  // development override (A/B)
    return v ? std::atoi(v) : 1;
  }();
  return env != 0 && Jmax <= 2 && N <= kBetaCarryMaxN;
}

int gene_dyn_smem(int N, int Jmax) {
  if (Jmax > 2) return gene_sweep_smem_bytes(N, Jmax);
  // the carried exps take the group-sum rows: N + 2 ceil(N/2) >= 2N
  return gene_sweep_smem_bytes(N, beta_carry_ok(N, Jmax) ? (N + 1) / 2 : 0);
}

int gene_sweep_smem_bytes(int N, int Jmax) {
  // lp [N][B] and the group sums [2 Jmax][B]; at least kGeneThreads / 32
  // staging rows of kStage for the fused leaf sums
  const int rows = N + 2 * Jmax;
  const int stage_rows = 2 * (kGeneThreads / 32) * kStageEpi / kGeneThreads;  // paired leaf sums
  return (int)(sizeof(double) * (size_t)(rows > stage_rows ? rows : stage_rows) * kGeneThreads);
}

cudaError_t launch_eps_sweep(const SweepParams& p, int chains, long m_off,
                             cudaStream_t s) {
  dim3 grid((unsigned)((p.G + kGeneBlock - 1) / kGeneBlock), (unsigned)p.N, (unsigned)chains);
  if (p.xi_any)
    return launch_prio(eps_sweep_kernel<CMC_EPS_XI_MIN_BLOCKS>, grid, dim3(kGeneBlock), 0, s,
                       p.prio_eps, p, m_off);
  if (p.eps_solo)
    return launch_prio(eps_sweep_kernel<CMC_EPS_SOLO_MIN_BLOCKS>, grid, dim3(kGeneBlock), 0, s,
                       p.prio_eps, p, m_off);
  return launch_prio(eps_sweep_kernel<CMC_EPS_MIN_BLOCKS>, grid, dim3(kGeneBlock), 0, s,
                     p.prio_eps, p, m_off);
}

template <int JR, bool XI>
static cudaError_t raise_smem(int dyn, int optin, int* total) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, gene_sweep_kernel<JR, XI, 3>);
  if (e != cudaSuccess) return e;
  *total = (int)fa.sharedSizeBytes + dyn;
  if (*total > optin) return cudaSuccess;  // the caller reports CMC_ERR_CONFIG
  if (dyn > fa.maxDynamicSharedSizeBytes) {
    const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
    if ((e = cudaFuncSetAttribute(gene_sweep_kernel<JR, XI, 3>, attr, dyn)) != cudaSuccess ||
        (e = cudaFuncSetAttribute(gene_sweep_kernel<JR, XI, 1>, attr, dyn)) != cudaSuccess)
      return e;
    e = cudaFuncSetAttribute(gene_sweep_kernel<JR, XI, 2>, attr, dyn);
  }
  return e;
}

// The attribute is per device: every engine sets it on its own device when
// it allocates (ensure_device), for the one gene kernel variant it launches,
// under one process-wide lock so engines of one device (loopback ranks)
// only ever raise it.  *total = static + dynamic bytes per block.
cudaError_t configure_gene_kernels(int N, int Jmax, int xi_any, int* total) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) !=
      cudaSuccess)
    return e;
  const int jr = Jmax <= 2;
  const int dyn = gene_dyn_smem(N, Jmax);
  if (jr) return xi_any ? raise_smem<2, true>(dyn, optin, total) : raise_smem<2, false>(dyn, optin, total);
  return xi_any ? raise_smem<0, true>(dyn, optin, total) : raise_smem<0, false>(dyn, optin, total);
}

template <int JR, bool XI>
static cudaError_t launch_gene_sweep_t(const SweepParams& p, int chains, long m_off,
                                       cudaStream_t s, int phase) {
  const int smem = gene_dyn_smem(p.N, p.Jmax);
  dim3 grid((unsigned)((p.G + kGeneThreads - 1) / kGeneThreads), (unsigned)chains);
  if (phase == 1)
    return launch_prio(gene_sweep_kernel<JR, XI, 1>, grid, dim3(kGeneThreads), smem, s,
                       p.prio_gene, p, m_off);
  if (phase == 2)
    return launch_prio(gene_sweep_kernel<JR, XI, 2>, grid, dim3(kGeneThreads), smem, s,
                       p.prio_gene, p, m_off);
  return launch_prio(gene_sweep_kernel<JR, XI, 3>, grid, dim3(kGeneThreads), smem, s,
                     p.prio_gene, p, m_off);
}

cudaError_t launch_gene_sweep(const SweepParams& p, int chains, long m_off,
                              cudaStream_t s, int phase) {
  if (p.xi_any) {
    if (p.Jmax <= 2) return launch_gene_sweep_t<2, true>(p, chains, m_off, s, phase);
    return launch_gene_sweep_t<0, true>(p, chains, m_off, s, phase);
  }
  if (p.Jmax <= 2) return launch_gene_sweep_t<2, false>(p, chains, m_off, s, phase);
  return launch_gene_sweep_t<0, false>(p, chains, m_off, s, phase);
}

// Layout transposes for state/output transfer: SoA [K][G] <-> the
// reference's AoS [G][K], through a 32-gene shared tile so both sides are
// coalesced (the host then moves one contiguous block).
__global__ void soa_to_aos_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                  long G, int K) {
  __shared__ double tile[32][65];
  const long g0 = (long)blockIdx.x * 32;
  for (int k0 = 0; k0 < K; k0 += 64) {
    const int kn = min(64, K - k0);
    for (int i = threadIdx.x; i < 32 * kn; i += blockDim.x) {
      const int k = i / 32, j = i % 32;
      if (g0 + j < G) tile[j][k] = src[(size_t)(k0 + k) * G + g0 + j];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * kn; i += blockDim.x) {
      const int j = i / kn, k = i % kn;
      if (g0 + j < G) dst[(size_t)(g0 + j) * K + k0 + k] = tile[j][k];
    }
    __syncthreads();
  }
}

__global__ void aos_to_soa_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                  long G, int K) {
  __shared__ double tile[32][65];
  const long g0 = (long)blockIdx.x * 32;
  for (int k0 = 0; k0 < K; k0 += 64) {
    const int kn = min(64, K - k0);
    for (int i = threadIdx.x; i < 32 * kn; i += blockDim.x) {
      const int j = i / kn, k = i % kn;
      if (g0 + j < G) tile[j][k] = src[(size_t)(g0 + j) * K + k0 + k];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * kn; i += blockDim.x) {
      const int k = i / 32, j = i % 32;
      if (g0 + j < G) dst[(size_t)(k0 + k) * G + g0 + j] = tile[j][k];
    }
    __syncthreads();
  }
}

cudaError_t launch_transpose(const double* src, double* dst, long G, int K, bool to_aos,
                             cudaStream_t s) {
  if (G <= 0 || K <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((G + 31) / 32);
  if (to_aos)
    soa_to_aos_kernel<<<blocks, 256, 0, s>>>(src, dst, G, K);
  else
    aos_to_soa_kernel<<<blocks, 256, 0, s>>>(src, dst, G, K);
  return cudaGetLastError();
}

cudaError_t launch_xi_sweep(const SweepParams& p, int chains, long m_off,
                            cudaStream_t s) {
  dim3 grid((unsigned)((p.G + kGeneBlock - 1) / kGeneBlock), (unsigned)p.L, (unsigned)chains);
  // parking pays for the heavy-tailed horseshoe loops only (A/B on B200,
  // DESIGN.md section 4): horseshoe 1.024 -> 0.950 ms per 4-chain sweep,
  // t 0.523 -> 0.548 with it
  bool hs = false;
  for (int l = 0; l < p.L; ++l) hs |= p.xi_fam[l] == CMC_PRIOR_HORSESHOE;
  static const int force = [] {  // development override (A/B): 1 park always, 0 never
    const char* v = std::getenv("CMC_XI_PARK");
    return v ? std::atoi(v) : -1;
  }();
  if (force >= 0) hs = force != 0;
  if (hs) return launch_prio(xi_park_kernel, grid, dim3(kGeneBlock), 0, s, p.prio_gene, p, m_off);
  return launch_prio(xi_sweep_kernel, grid, dim3(kGeneBlock), 0, s, p.prio_gene, p, m_off);
}

cudaError_t launch_leaf_a(const SweepParams& p, int chains, long m_off,
                          cudaStream_t s) {
  const int Q = leaf_q_a(p.L, p.xi_any);
  const int threads = 32 * (Q < kTailWarps ? Q : kTailWarps);
  dim3 grid((unsigned)p.n_leaves_local, (unsigned)chains);
  if (p.xi_any)
    return launch_prio(leaf_a_kernel<true>, grid, dim3(threads < 64 ? 64 : threads), 0, s,
                       p.prio_tail, p, m_off);
  return launch_prio(leaf_a_kernel<false>, grid, dim3(threads < 64 ? 64 : threads), 0, s,
                     p.prio_tail, p, m_off);
}

cudaError_t launch_hyper_a(const SweepParams& p, int chains, long m_off,
                           cudaStream_t s) {
  const int Q = leaf_q_a(p.L, p.xi_any);
  const int threads = 32 * (Q < kTailWarps ? Q : kTailWarps);
  if (p.xi_any)
    return launch_prio(hyper_a_kernel<true>, dim3(chains), dim3(threads < 64 ? 64 : threads), 0, s,
                       p.prio_tail, p, m_off);
  return launch_prio(hyper_a_kernel<false>, dim3(chains), dim3(threads < 64 ? 64 : threads), 0,
                     s, p.prio_tail, p, m_off);
}

cudaError_t launch_leaf_b(const SweepParams& p, int chains, long m_off,
                          cudaStream_t s) {
  const int threads = 32 * (p.L > 1 ? p.L : 1);
  dim3 grid((unsigned)p.n_leaves_local, (unsigned)chains);
  if (p.xi_any)
    return launch_prio(leaf_b_kernel<true>, grid, dim3(threads < 32 ? 32 : threads), 0, s,
                       p.prio_tail, p, m_off);
  return launch_prio(leaf_b_kernel<false>, grid, dim3(threads < 32 ? 32 : threads), 0, s,
                     p.prio_tail, p, m_off);
}

cudaError_t launch_hyper_b(const SweepParams& p, int chains, long m_off,
                           cudaStream_t s) {
  return launch_prio(hyper_b_kernel, dim3(chains), dim3(32 * p.L), 0, s, p.prio_tail, p, m_off);
}

cudaError_t launch_gene_contrast(const SweepParams& p, int chains, long m_off,
                                 cudaStream_t s) {
  dim3 grid((unsigned)((p.G + 255) / 256), (unsigned)chains);
  return launch_prio(gene_contrast_kernel, grid, dim3(256), 0, s, p.prio_tail, p, m_off);
}

cudaError_t launch_fastmath_setup(cudaStream_t s) {
  fastmath_setup_kernel<<<1, 32, 0, s>>>();
  return cudaGetLastError();
}

cudaError_t launch_fill(double* p, size_t n, double v, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const size_t blocks = std::min<size_t>((n + 255) / 256, 148 * 16);
  fill_kernel<<<(unsigned)blocks, 256, 0, s>>>(p, n, v);
  return cudaGetLastError();
}

cudaError_t launch_advance(long* d_m, long by, cudaStream_t s) {
  advance_kernel<<<1, 1, 0, s>>>(d_m, by);
  return cudaGetLastError();
}

cudaError_t launch_compute_A(const double* y, const double* X, double* A,
                             int G, int N, int L, cudaStream_t s) {
  compute_A_kernel<<<(G + 255) / 256, 256, 0, s>>>(y, X, A, G, N, L);
  return cudaGetLastError();
}

}  // namespace cmc

// ------------------------------------------------------ post-run diagnostics
namespace cmc {
namespace {

// gelman_rhat (P:src/diagnostics.cpp:11-37) and the pooled estimate with
// its credible interval (pool_moments / credible_interval, P:src/io.cpp:
// 483-505, P:src/diagnostics.cpp:46-57) for one parameter row.
__device__ void diag_row(const DiagParams& d, long r, const double* means,
                         const double* meansqs) {
  const int C = d.C;
  const double Md = (double)d.M;
  double grand = 0.0;
  for (int c = 0; c < C; ++c) grand += means[c];
  grand /= (double)C;
  double B = 0.0, W = 0.0;
  for (int c = 0; c < C; ++c) {
    const double dm = means[c] - grand;
    B += dm * dm;
    const double v = meansqs[c] - means[c] * means[c];
    const double var = (0.0 < v) ? v : 0.0;  // std::max(0.0, v)
    W += (Md / (Md - 1.0)) * var;
  }
  B *= Md / (double)(C - 1);
  W /= (double)C;
  int flags = 0;
  double rh = 1.0;
  if (!(W > 0.0)) {
    flags |= 1;
  } else {
    rh = sqrt(1.0 + (B / W - 1.0) / Md);
  }
  if ((flags & 1) || rh < 1.1) flags |= 2;
  double pm = 0.0, pms = 0.0;
  for (int c = 0; c < C; ++c) {
    pm += means[c];
    pms += meansqs[c];
  }
  pm /= (double)C;
  pms /= (double)C;
  const double v = pms - pm * pm;
  const double sd = sqrt((0.0 < v) ? v : 0.0);
  const double slack = 1e-9 * ((1.0 < fabs(pms)) ? fabs(pms) : 1.0);
  double var = v;
  if (var < -slack) flags |= 4;
  if (var < 0.0) var = 0.0;
  const double half = d.z * sqrt(var);
  d.rhat[r] = rh;
  d.mean[r] = pm;
  d.sd[r] = sd;
  d.lo[r] = pm - half;
  d.hi[r] = pm + half;
  d.flags[r] = flags;
}

__global__ void diag_rows_kernel(const DiagParams d) {
  const long r = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int L = d.L;
  const long R = 2 + 2 * L + d.G * (L + 1);
  if (r >= R) return;
  double means[32], meansqs[32];
  const int C = d.C;
  const size_t G = (size_t)d.G;
  for (int c = 0; c < C; ++c) {
    if (r < 2 + 2 * L) {
      means[c] = d.hyper[c].acc[0][r];
      meansqs[c] = d.hyper[c].acc[1][r];
    } else if (r < 2 + 2 * L + d.G * L) {
      const long k = r - 2 - 2 * L, g = k / L, l = k % L;
      const double* a = d.acc_beta + (size_t)c * 4 * L * G + (size_t)l * G + g;
      means[c] = a[0];
      meansqs[c] = a[(size_t)L * G];
    } else {
      const long g = r - 2 - 2 * L - d.G * L;
      const double* a = d.acc_gam + (size_t)c * 4 * G + g;
      means[c] = a[0];
      meansqs[c] = a[G];
    }
  }
  diag_row(d, r, means, meansqs);
}

// effective_sample_size for one retained column (P:src/diagnostics.cpp:
// 80-114): one warp; each lane computes whole lag autocovariances in the
// reference's serial order, lane 0 runs the Geyer initial-positive,
// monotone pair scan.
__global__ void diag_ess_kernel(const DiagParams d) {
  // lags are computed 64 at a time (two per lane) and lane 0 runs the
  // Geyer scan over each batch, stopping where the reference stops: cost
  // O(M x cutoff) like avg_autocov on demand, and O(1) shared memory
  __shared__ double lagb[64];
  __shared__ double mu[32];
  const long col = blockIdx.x;
  const int lane = threadIdx.x;
  const long M = d.n_rows;
  const int C = d.C;
  if (M < 4) {
    if (lane == 0) {
      d.ess[col] = 0.0;
      d.ess_status[col] = 1;
    }
    return;
  }
  auto x = [&](int c, long i) {
    return d.samples[((size_t)c * d.n_cols + col) * M + i];
  };
  if (lane < C) {
    double s = 0.0;
    for (long i = 0; i < M; ++i) s += x(lane, i);
    mu[lane] = s / (double)M;
  }
  __syncwarp();
  // avg_autocov(t), P:src/diagnostics.cpp: chains in order, biased 1/M
  auto autocov = [&](long t) {
    double total = 0.0;
    for (int c = 0; c < C; ++c) {
      double s = 0.0;
      for (long i = 0; i + t < M; ++i) s += (x(c, i) - mu[c]) * (x(c, i + t) - mu[c]);
      total += s / (double)M;
    }
    return total / (double)C;
  };
  double c0 = 0.0, tau = 0.0, prev = INFINITY;
  int status = -1;  // lane 0: -1 running, 0 ok (scan ended), 2 degenerate
  for (long base = 0; base < M; base += 64) {
    for (int j = lane; j < 64; j += 32) {
      const long t = base + j;
      lagb[j] = t < M ? autocov(t) : 0.0;
    }
    __syncwarp();
    if (lane == 0) {
      if (base == 0) {
        c0 = lagb[0];
        if (!(c0 > 0.0)) status = 2;
      }
      for (int j = 0; status < 0 && j < 64; j += 2) {
        const long k2 = base + j;  // 2k
        if (!(k2 + 1 < M)) {
          status = 0;
          break;
        }
        const double re = lagb[j] / c0;
        const double ro = lagb[j + 1] / c0;
        double pair = re + ro;
        if (pair <= 0.0) {
          status = 0;
          break;
        }
        pair = (prev < pair) ? prev : pair;  // std::min(pair, prev)
        prev = pair;
        tau += pair;
      }
    }
    const int st = __shfl_sync(0xffffffffu, status, 0);
    __syncwarp();
    if (st >= 0) break;
  }
  if (lane != 0) return;
  if (status == 2) {
    d.ess[col] = 0.0;
    d.ess_status[col] = 2;
    return;
  }
  const double total = (double)C * (double)M;
  tau = 2.0 * tau - 1.0;
  if (tau < 1.0) tau = 1.0;
  d.ess[col] = total / tau;
  d.ess_status[col] = 0;
}

}  // namespace

cudaError_t launch_diagnostics(const DiagParams& d, cudaStream_t s) {
  const long R = 2 + 2 * d.L + d.G * (d.L + 1);
  diag_rows_kernel<<<(unsigned)((R + 127) / 128), 128, 0, s>>>(d);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || d.n_cols == 0) return e;
  diag_ess_kernel<<<(unsigned)d.n_cols, 32, 0, s>>>(d);
  return cudaGetLastError();
}

}  // namespace cmc
