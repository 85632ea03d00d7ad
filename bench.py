#!/usr/bin/env python
"""Benchmark: MCMC gene-iterations/sec of the B200 Gibbs sweep.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step is one monitored Gibbs sweep (iterate + run_chain's Welford monitors,
per-gene heterosis contrast and thinning, P:src/engine.cpp:409-447) of every
chain.  Workloads (BASELINE.json):

* N = 1 (default): configs[1], Paschold-shaped synthetic data, G = 39,656,
  N = 16 samples, L = 5 (heterosis16x5), Normal beta prior, 4 chains (the
  reference RunConfig default), widths tuned by 200 burn-in sweeps.
* N > 1 (torchrun): configs[3], G = 1,000,000 genes in total, sharded over
  the ranks (strong scaling) with an NCCL all-gather of the leaf partial
  sums per sweep.  The N = 1 line carries the 1-GPU G = 1M point too
  (other_configs), so the scaling curve has its 1-GPU anchor.

Inputs are the reference's own generate() (P:src/simulate.cpp:28-90) on
both arms: the product's cmc_simulate is bit-identical to it
(tests/test_abi.py), and the reference arm calls the compiled reference.

--impl reference times the UNMODIFIED reference CPU sampler (compiled from
/root/reference into oracle/_ref) on all host threads on the same workload;
that arm maps only oracle/ libraries.
"""
import argparse
import json
import os
import subprocess
import sys
import time
from ctypes import byref, c_double

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

THETA = [2.5, 0.2, 0.2, 0.0, 0.1]
SIGMA = [0.4, 0.25, 0.25, 0.15, 0.2]
NU, TAU, DATA_SEED = 8.0, 0.7, 1
PAPER_K20 = 2.27e6  # fbseqCUDA on a K20, PAPER.md:371 (different code, context only)
WORKLOADS = {
    "paschold": ("paschold_G39656_N16_L5_heterosis16x5", 39656, 16),
    "g1m": ("G1000000_N16_L5_heterosis16x5", 1_000_000, 16),
    "g200k_n64": ("G200000_N64_L5_heterosis16x5", 200_000, 64),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto"] + list(WORKLOADS))
    ap.add_argument("--chains", type=int, default=4)
    ap.add_argument("--burnin", type=int, default=200)
    ap.add_argument("--e2e-burnin", type=int, default=2000)      # reference RunConfig default
    ap.add_argument("--e2e-iterations", type=int, default=4000)  # reference RunConfig default
    ap.add_argument("--e2e-reps", type=int, default=3)  # complete runs; the fastest is reported
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-min-sweeps", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-xi", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    # test hook: run the sharded (N > 1) code path as a 1-rank NCCL clique
    # (process group, uid broadcast, shard, collectives, stall exchange)
    ap.add_argument("--force-shard", action="store_true")
    return ap.parse_args()


def workload(a, world):
    key = a.workload
    if key == "auto":
        key = "paschold" if world == 1 and not getattr(a, "force_shard", False) else "g1m"
    return (key,) + WORKLOADS[key]


def problem(G, N):
    """The product's generator: bit-identical to the reference's generate()."""
    from paper_1606_06659_b200 import SimSpec, builtin_design, generate
    X = builtin_design("heterosis16x5", N)
    counts = generate(SimSpec(G=G, N=N, X=X, nu=NU, tau=TAU, theta=THETA, sigma=SIGMA,
                              seed=DATA_SEED)).counts
    return counts, X, np.zeros(N)


def bytes_per_gene_iter(N, L, n_gene_contrasts):
    """Minimum HBM bytes of one monitored gene-iteration:
    reads y 4N, eps 8N, w_eps 8N, gamma 8, w_gamma 8, beta 8L, w_beta 8L;
    writes eps 8N, gamma 8, beta 8L; compensated-Welford monitors (4 doubles
    read + written) for N+L+1 scalars; 16 B per per-gene contrast."""
    return 92 * N + 88 * L + 88 + 16 * n_gene_contrasts


def phase_bytes(N, L, n_gene_contrasts):
    """B_mon split by the kernel that moves it: eps (y, eps, w_eps, eps
    monitors: 92N), gene (gamma, w_gamma, beta, w_beta, their monitors and
    the contrasts: 88L + 88 + 16 K_c)."""
    return {"eps": 92 * N, "gene": 88 * L + 88 + 16 * n_gene_contrasts}


def nproc():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


HETEROSIS = [([("beta_col", 1, 2.0), ("beta_col", 3, 1.0)], 0.0),
             ([("beta_col", 2, 2.0), ("beta_col", 3, 1.0)], 0.0)]


def reference_rate(G, N, burnin, sweeps=None, seconds=None, workers=None, chains=1,
                   min_sweeps=3):
    """The UNMODIFIED reference (oracle/_ref): generate() for the inputs,
    GibbsEngine::iterate + run_chain's monitors for the timing, `chains`
    chains one after another as run() does, each after `burnin` untimed
    burn-in sweeps on all host threads, its monitored sweeps timed on
    `workers` threads (all by default).  Only oracle/ libraries are used.
    Returns (gene-iter/s, threads, sweeps per chain, seconds)."""
    import oracle
    from paper_1606_06659_b200 import _abi   # ctypes structs only, no library load
    if not oracle.ref_available():
        raise RuntimeError("oracle/_ref/libcountmc_ref.so missing")
    all_threads = nproc()
    threads = workers or all_threads
    counts, X = oracle.ref_generate(G, N, NU, TAU, THETA, SIGMA, DATA_SEED)
    h = np.zeros(N)
    cfg = _abi.make_config(chains=chains, burnin=burnin, iterations=10 ** 6, thin=20, seed=7,
                           save_genes=20, workers=threads)
    eng = oracle.RefEngine(counts, X, h, cfg, contrasts=[HETEROSIS], workers=threads)
    if sweeps is None:
        probe = eng.bench(threads, burnin, 3, burn_workers=all_threads)
        sweeps = max(min_sweeps, int(seconds / max(probe / 3, 1e-6) / chains))
    secs = eng.bench(threads, burnin, sweeps, burn_workers=all_threads, chains=chains)
    return chains * G * sweeps / secs, threads, sweeps, secs


class Clocks:
    """nvidia-smi sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)
        self.proc.terminate()
        out, _ = self.proc.communicate()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def run_reference(a, rank, world):
    """--impl reference: the reference CPU sampler on this box's host cores,
    on this arm's workload (rank 0 only)."""
    if rank != 0:
        return
    key, wname, G, N = workload(a, world)
    big = G * N > 2_000_000
    B = 100 if big else a.burnin + a.warmup
    chains = 1 if big else a.chains
    sweeps = max(a.steps, 3) if big else max(a.steps, a.ref_min_sweeps)
    rate, threads, sweeps, secs = reference_rate(G, N, B, sweeps=sweeps, chains=chains)
    sample = (f"{chains} chain(s) x {sweeps} monitored sweeps at G={G} N={N} (chains in "
              f"sequence, as run()), each after {B} burn-in sweeps; reference iterate() + "
              f"run_chain monitors + heterosis contrast, workers={threads}, {cpu_model()}")
    line = {
        "impl": "reference", "metric": "MCMC gene-iterations/sec", "value": rate,
        "unit": "gene-iter/s", "n_gpus": world, "steps": sweeps * chains, "warmup": a.warmup,
        "ms_per_step": secs / (sweeps * chains) * 1e3, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the reference's own generate() (heterosis16x5, seed 1)",
        "config": {"workload": wname, "G": G, "N": N, "L": 5, "chains": chains, "burnin": B,
                   "contrasts": "heterosis (per gene)", "sampler": "slice_faithful",
                   "threads": threads,
                   "steps_note": f"a step is one chain-sweep; {sweeps} sweeps per chain are "
                                 f"timed (at least {a.ref_min_sweeps} at G <= 100k) whatever "
                                 f"--steps asks ({a.steps})"},
        "cpu_baseline": {"value": rate, "unit": "gene-iter/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": rate, "unit": "gene-iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(a, rank, world, local_rank):
    import torch
    import paper_1606_06659_b200 as pkg
    from paper_1606_06659_b200 import (CountMatrix, GibbsEngine, ModelSpec, RunConfig,
                                       heterosis_contrast)
    from paper_1606_06659_b200._abi import CMC_PHASES, PHASE_NAMES, CmcError
    dist = world > 1 or a.force_shard
    torch.cuda.set_device(local_rank)
    key, wname, G, N = workload(a, world)
    counts, X, h = problem(G, N)
    C, B, W, K = a.chains, a.burnin, a.warmup, a.steps
    prof_reps = 5
    n_probe_max = 20000
    # iterations cover warm-up, the clock probe (below), the timed steps and
    # the profile reps; monitors run on all of them like run_chain's
    cfg = RunConfig(chains=C, burnin=B, iterations=W + n_probe_max + 2 * K + prof_reps,
                    thin=20, seed=7, save_genes=20)
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg,
                      contrasts=[heterosis_contrast()], device=local_rank)

    def shard(e):
        import torch.distributed as td
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(GibbsEngine.nccl_unique_id()),
                                       dtype=torch.uint8))
        td.broadcast(uid, 0)
        e.shard(rank, world, bytes(uid.cpu().numpy().tobytes()))

    if dist:
        shard(eng)
    lib, hd, err = eng._lib, eng.handle, CmcError()

    def ok(rc):
        if rc:
            raise RuntimeError(err.msg.decode())

    ok(lib.cmc_engine_begin(hd, byref(err)))
    stream = torch.cuda.ExternalStream(lib.cmc_engine_stream(hd))
    # burn-in (tuning active, no monitors), timed separately:
    # sweeps 1..5 start from w_init = 1 (the divergent-slice-loop proxy,
    # config 3); the next 50 include the one-time capture of the sweep graph;
    # the rest is the steady burn-in rate.  The graphs of the first-sweeps
    # call and of the rest are captured up front (cmc_engine_prepare).
    nb0 = min(5, B)
    nb1 = min(50, B - nb0)
    for n_ in (nb0, B - nb0 - nb1, W, K):
        if n_ > 0:
            ok(lib.cmc_engine_prepare(hd, n_, byref(err)))
    b0, b1, b2, b3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
    b0.record(stream)
    ok(lib.cmc_engine_sweeps(hd, 1, 1 + nb0, byref(err)))
    b1.record(stream)
    ok(lib.cmc_engine_sweeps(hd, 1 + nb0, 1 + nb0 + nb1, byref(err)))
    b2.record(stream)
    ok(lib.cmc_engine_sweeps(hd, 1 + nb0 + nb1, B + 1, byref(err)))    # rest of burn-in
    b3.record(stream)
    w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0.record(stream)
    ok(lib.cmc_engine_sweeps(hd, B + 1, B + 1 + W, byref(err)))  # warm-up monitored steps
    w1.record(stream)
    ok(lib.cmc_engine_sync(hd, byref(err)))
    warm_ms = w0.elapsed_time(w1) / max(W, 1)
    burn_first_ms, burn_cap_ms, burn_rest_ms = (b0.elapsed_time(b1), b1.elapsed_time(b2),
                                                b2.elapsed_time(b3))
    n_rest = B - nb0 - nb1
    Cg = C * G
    burnin = {"value": Cg * n_rest / (burn_rest_ms * 1e-3) if n_rest else None,
              "unit": "gene-iter/s", "sweeps": B,
              "ms_per_sweep": burn_rest_ms / n_rest if n_rest else None,
              "first_sweeps": nb0, "first_ms_per_sweep": burn_first_ms / max(nb0, 1),
              "graph_capture_chunk_ms": burn_cap_ms,
              "note": "burn-in sweeps (tuning on, no monitors), device-timed: value and "
                      "ms_per_sweep over sweeps 56..B; first_* are sweeps 1..5 from w_init=1 "
                      "(wide, divergent slice loops); graph_capture_chunk_ms is sweeps 6..55 "
                      "including the one-time capture of the 50-sweep graph (the other "
                      "graphs are captured before the timed calls)"}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    # clocks are sampled under load: untimed monitored sweeps keep the GPU busy
    # for ~0.4 s right before the timed region, inside the sampler's window.
    # They run in calls of K sweeps, so the K-sweep CUDA graph the timed call
    # replays is captured here, outside the timed region.
    n_probe = max(K, min(n_probe_max, int(400.0 / max(warm_ms, 1e-3)) // K * K))
    if dist:
        # every rank must run the same sweeps (each sweep's all-gathers are
        # collective): rank 0's probe length for all
        t = torch.tensor([n_probe], device="cuda", dtype=torch.int64)
        torch.distributed.broadcast(t, 0)
        n_probe = int(t.item())
    m0 = B + 1 + W + n_probe
    clocks = Clocks(local_rank)
    clocks.start()
    time.sleep(0.1)  # nvidia-smi start-up
    for mb in range(B + 1 + W, m0, K):
        ok(lib.cmc_engine_sweeps(hd, mb, mb + K, byref(err)))
    ok(lib.cmc_engine_sync(hd, byref(err)))
    torch.cuda.synchronize()
    if dist:
        torch.distributed.barrier()
    e0.record(stream)
    ok(lib.cmc_engine_sweeps(hd, m0, m0 + K, byref(err)))
    e1.record(stream)
    ok(lib.cmc_engine_sync(hd, byref(err)))
    torch.cuda.synchronize()
    if dist:
        torch.distributed.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = Cg * K / (ms * 1e-3)
    ms_step = ms / K
    # the sweep kernels of every lane, plus one iteration-advance kernel per
    # graph replay (K // 50 full 50-sweep graphs and one of the remainder)
    graphs = K // 50 + (1 if K % 50 else 0)
    launches = K * lib.cmc_engine_launches_per_sweep(hd) + graphs

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    G_local = G
    if dist:
        from ctypes import c_long
        lo, hi = c_long(), c_long()
        lib.cmc_shard_bounds(G, rank, world, byref(lo), byref(hi))
        G_local = hi.value - lo.value
    roofline = None
    bpg = bytes_per_gene_iter(N, 5, 1)
    per_step = C * G_local * bpg
    achieved = per_step / (ms_step * 1e-3) / 1e9
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "traffic": None,
        "kernel": "the whole sweep (eps + gene + tail kernels of both chain lanes, one "
                  "graph replay): algorithmic bytes per step / ms_per_step",
        "algorithmic_bytes_per_step": per_step, "bytes_per_gene_iter": bpg,
        "peak_source": ("MEASURED_PEAKS.json hbm_gbs (burst)" if "hbm_gbs" in peaks
                        else "fallback 6.65 TB/s"),
    }
    if not dist:
        # per kernel, each phase alone for all chains (serialised; their sum
        # exceeds ms_per_step because the graph overlaps lanes and streams)
        ph = (c_double * CMC_PHASES)()
        ok(lib.cmc_engine_profile_phases(hd, m0 + K, prof_reps, ph, byref(err)))
        pb = phase_bytes(N, 5, 1)
        kern = {}
        for i, name in enumerate(PHASE_NAMES):
            if ph[i] <= 0.0005:
                continue
            kern[name] = {"ms_alone": ph[i]}
            if name in pb:
                b = C * G * pb[name]
                kern[name].update(algorithmic_bytes=b, achieved_gbs=b / (ph[i] * 1e-3) / 1e9,
                                  frac=b / (ph[i] * 1e-3) / 1e9 / peak)
        kern["sum_ms_alone"] = sum(ph[i] for i in range(CMC_PHASES))
        roofline["kernels"] = kern
        # DRAM traffic of a whole 50-sweep graph replay (ncu --graph-profiling
        # graph: write-back included), per sweep, from the committed capture
        tpath = os.path.join(ROOT, "profiles", "graph_traffic.json")
        if os.path.exists(tpath):
            tj = json.load(open(tpath))
            if tj.get("chains") == C and tj.get("G") == G and tj.get("N") == N:
                roofline["traffic"] = tj.get("dram_bytes_per_sweep")
                roofline["traffic_source"] = tj.get("source")
                if tj.get("fp64_pipe"):
                    roofline["fp64_pipe"] = tj["fp64_pipe"]
        # the bound the sweep sits on: warp-instruction issue
        ipath = os.path.join(ROOT, "profiles", "sweep_instructions.json")
        if os.path.exists(ipath):
            ij = json.load(open(ipath))
            if ij.get("chains") == C and ij.get("G") == G and ij.get("N", 16) == N:
                mhz = (clk or {}).get("sm_mhz") or 1965.0
                ipeak = 148 * 4 * mhz * 1e6          # 1 warp-instruction / scheduler / clock
                iach = ij["warp_inst_per_sweep"] / (ms_step * 1e-3)
                roofline["issue_roofline"] = {
                    "bound": "issue", "achieved": iach, "peak": ipeak, "unit": "warp-inst/s",
                    "frac": iach / ipeak, "warp_inst_per_sweep": ij["warp_inst_per_sweep"],
                    "source": ij.get("source"),
                    "note": "ncu instruction count of the sweep kernels per 4-chain sweep over "
                            "the live ms_per_step; peak = 148 SMs x 4 schedulers x SM clock"}
        roofline["note"] = ("the sweep is issue/latency bound, not HBM bound (issue_roofline; "
                            "DESIGN.md §5)")
    del eng
    torch.cuda.synchronize()

    # BASELINE configs[1] names Laplace priors, configs[2] t and horseshoe:
    # the xi extension (not in the reference; parity unpinned)
    # timed the same way on the same data.  The headline stays the normal
    # prior, the only model the reference (and so the reference arm) has.
    xi_rates = None
    if not dist and not a.no_xi and key == "paschold":
        xi_rates = {}
        from paper_1606_06659_b200 import PriorConfig
        for name in ("laplace", "t", "horseshoe"):
            spec = ModelSpec(X, h, PriorConfig(beta_prior=[name], t_df=3.0))
            ex = GibbsEngine(CountMatrix(counts), spec,
                             RunConfig(chains=C, burnin=B, iterations=W + 2 * K, thin=20,
                                       seed=7, save_genes=20),
                             contrasts=[heterosis_contrast()], device=local_rank)
            lx, hx = ex._lib, ex.handle
            ok(lx.cmc_engine_begin(hx, byref(err)))
            ok(lx.cmc_engine_prepare(hx, nb0, byref(err)))
            sx = torch.cuda.ExternalStream(lx.cmc_engine_stream(hx))
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(sx)
            ok(lx.cmc_engine_sweeps(hx, 1, 1 + nb0, byref(err)))
            f1.record(sx)
            ok(lx.cmc_engine_sweeps(hx, 1 + nb0, B + 1 + W, byref(err)))
            ok(lx.cmc_engine_sweeps(hx, B + 1 + W, B + 1 + W + K, byref(err)))  # K graph
            ok(lx.cmc_engine_sync(hx, byref(err)))
            x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            x0.record(sx)
            ok(lx.cmc_engine_sweeps(hx, B + 1 + W + K, B + 1 + W + 2 * K, byref(err)))
            x1.record(sx)
            ok(lx.cmc_engine_sync(hx, byref(err)))
            torch.cuda.synchronize()
            xms = x0.elapsed_time(x1)
            xi_rates[name] = {"value": Cg * K / (xms * 1e-3), "ms_per_step": xms / K,
                              "first_ms_per_sweep": f0.elapsed_time(f1) / max(nb0, 1)}
            del ex
        xi_rates["note"] = ("beta_gl ~ N(theta_l, sigma_l^2 xi_gl) with a xi slice step per "
                            "(gene, column); t with k = 3; same data, chains, burn-in and "
                            "device timing as value; extension, not in the reference")

    # BASELINE configs 4 and 5 on this GPU (parity cases, not the headline),
    # with the reference CPU sampler beside each (rank 0, N = 1)
    other = None
    if not dist and not a.no_other_configs:
        other = {}
        for okey in ("g1m", "g200k_n64"):
            oname, Gx, Nx = WORKLOADS[okey]
            cx, Xx, hx_ = problem(Gx, Nx)
            ex = GibbsEngine(CountMatrix(cx), ModelSpec(Xx, hx_),
                             RunConfig(chains=C, burnin=100, iterations=100, thin=20, seed=7,
                                       save_genes=20),
                             contrasts=[heterosis_contrast()], device=local_rank)
            lx, hdx = ex._lib, ex.handle
            ok(lx.cmc_engine_begin(hdx, byref(err)))
            ok(lx.cmc_engine_sweeps(hdx, 1, 106, byref(err)))
            ok(lx.cmc_engine_sweeps(hdx, 106, 126, byref(err)))   # captures the 20-sweep graph
            ok(lx.cmc_engine_sync(hdx, byref(err)))
            sx = torch.cuda.ExternalStream(lx.cmc_engine_stream(hdx))
            y0, y1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            y0.record(sx)
            ok(lx.cmc_engine_sweeps(hdx, 126, 146, byref(err)))
            y1.record(sx)
            ok(lx.cmc_engine_sync(hdx, byref(err)))
            torch.cuda.synchronize()
            yms = y0.elapsed_time(y1) / 20
            bx = C * Gx * bytes_per_gene_iter(Nx, 5, 1)
            other[okey] = {"workload": oname, "value": C * Gx / (yms * 1e-3),
                           "ms_per_step": yms, "chains": C,
                           "roofline_frac": bx / (yms * 1e-3) / 1e9 / peak}
            del ex, cx
            if not a.no_cpu_baseline:
                try:
                    r, thr, sw, _ = reference_rate(Gx, Nx, 100, sweeps=3)
                    other[okey]["cpu_baseline"] = {
                        "value": r, "unit": "gene-iter/s", "cores": thr, "kind": "reference",
                        "sample": f"1 chain x {sw} monitored sweeps after 100 burn-in sweeps, "
                                  f"workers={thr}, {cpu_model()}"}
                    other[okey]["ratio_vs_cpu"] = other[okey]["value"] / r
                except Exception as ex_:  # report, never fake
                    other[okey]["cpu_baseline"] = {"value": None, "sample": f"unavailable: {ex_}"}
        other["note"] = ("BASELINE configs 4 (G=1M, N=16; one GPU) and 5 (G=200k, N=64), "
                         "heterosis16x5, normal prior, 4 chains, 105 burn-in then 20 "
                         "device-timed monitored sweeps (one 20-sweep graph replay); "
                         "cpu_baseline: the reference on all host cores, 1 chain")

    # end to end through the public API from host arrays: create (H2D of
    # counts + initial states), run() (burn-in + iterations), all outputs D2H
    e2e = None
    if not a.no_e2e:
        E, BE = a.e2e_iterations, a.e2e_burnin
        cfg_e = RunConfig(chains=C, burnin=BE, iterations=E, thin=20, seed=7, save_genes=20)
        walls = []
        for _ in range(max(1, a.e2e_reps)):
            if dist:
                torch.distributed.barrier()
            t0 = time.perf_counter()
            eng2 = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg_e,
                               contrasts=[heterosis_contrast()], device=local_rank)
            if dist:
                shard(eng2)
            outs = eng2.run()
            t1 = time.perf_counter()
            wall = t1 - t0
            if dist:
                t = torch.tensor([wall], device="cuda", dtype=torch.float64)
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                wall = float(t.item())
            walls.append(wall)
            del eng2
        wall = min(walls)
        S, T, A = pkg.sizes(G, N, 5)
        h2d = counts.size * 8 + X.size * 8 + h.size * 8 + C * (S + 2 * T) * 8
        d2h = C * (4 * A * 8 + S * 8 + G * 8 + outs[0].samples.size * 8)
        e2e = {"value": Cg * (BE + E) / wall, "unit": "gene-iter/s",
               "h2d_bytes_per_step": h2d / (BE + E), "d2h_bytes_per_step": d2h / (BE + E),
               "accounting": "all sweeps: chains x G x (burn-in + monitored sweeps) / wall",
               "post_burnin_value": Cg * E / wall,
               "post_burnin_accounting": "BASELINE.md's strict form: chains x G x monitored "
                                         "sweeps / the whole wall (burn-in time charged too)",
               "wall_s": wall, "wall_s_all": walls, "sweeps": BE + E, "burnin": BE,
               "iterations": E,
               "note": "one GibbsEngine(...).run() with the reference's default RunConfig "
                       "(chains 4, burnin 2000, iterations 4000), host wall clock: host count "
                       "matrix in (H2D), every sweep, all ChainOutputs out (D2H).  value leads "
                       "with every sweep the call ran (a burn-in sweep costs what a monitored "
                       "one costs on both sides, and the reference arm's rate is per sweep); "
                       "post_burnin_value is the strict form.  An MCMC run has one input (the "
                       "counts) and one result (the ChainOutputs): the per-step byte figures "
                       "are run totals over the sweeps.  Fastest of e2e_reps complete runs "
                       "(max over ranks per run)"}

    if rank != 0:
        return
    cpu = None
    if not a.no_cpu_baseline and not dist:
        try:
            rate, threads, steps, secs = reference_rate(G, N, B + W, seconds=a.cpu_seconds,
                                                        min_sweeps=a.ref_min_sweeps)
            cpu = {"value": rate, "unit": "gene-iter/s", "cores": threads, "kind": "reference",
                   "sample": f"1 chain x {steps} monitored sweeps at G={G} after {B + W} "
                             f"burn-in sweeps, reference iterate() + run_chain monitors + "
                             f"heterosis contrast, workers={threads}, {cpu_model()}"}
            r1, _, s1, _ = reference_rate(G, N, B + W, seconds=a.cpu_seconds / 3, workers=1)
            cpu["single_core"] = {"value": r1, "cores": 1,
                                  "sample": f"{s1} monitored sweeps, workers=1 (burn-in on "
                                            f"all threads)"}
        except Exception as ex:  # report, never fake
            cpu = {"value": None, "unit": "gene-iter/s", "cores": nproc(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}
    line = {
        "metric": "MCMC gene-iterations/sec", "value": value, "unit": "gene-iter/s",
        "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong" if dist else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: the reference's generate() (heterosis16x5, seed 1; cmc_simulate "
                "is bit-identical to it), random-initialised chains",
        "config": {"workload": wname, "G": G, "G_per_gpu": G_local, "N": N, "L": 5,
                   "chains": C, "burnin": B, "thin": 20, "contrasts": "heterosis (per gene)",
                   "sampler": "slice_faithful", "prior": "normal (reference has no Laplace)",
                   "parallelism": f"gene-shard x{world} (NCCL all-gather of leaf sums)"
                                  if dist else "single GPU",
                   "timed": f"{K} sweeps in one cmc_engine_sweeps call, replayed from "
                            f"{graphs} CUDA graph launch(es)",
                   "l2": "inputs larger than L2: ~%.0f MB touched per sweep vs 126 MB L2"
                         % (per_step / 1e6 + G_local * N * 8 / 1e6)},
        "gpu_launches": launches,
        "clocks": dict(clk, probe_sweeps=n_probe,
                       note="nvidia-smi -lms 50 over ~0.4 s of untimed monitored sweeps "
                            "plus the timed region"),
        "burnin": burnin,
        "xi_priors": xi_rates,
        "other_configs": other,
        "e2e": e2e,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "paper_k20_ratio": value / PAPER_K20,
    }
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus and "WORLD_SIZE" in os.environ:
        print(f"warning: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    if world > 1 or a.force_shard:
        # NCCL init logging (nranks per communicator) for the driver's check;
        # set outright: an inherited NCCL_DEBUG=WARN would hide it
        # to stderr: stdout carries the one JSON line
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
        os.environ["NCCL_DEBUG_FILE"] = "/dev/stderr"
        print(f"[bench] rank {rank}: NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT (stderr)",
              file=sys.stderr)
        import torch
        import torch.distributed as td
        torch.cuda.set_device(local_rank)
        td.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_b200(a, rank, world, local_rank)
    finally:
        if world > 1 or a.force_shard:
            import torch.distributed as td
            td.destroy_process_group()


if __name__ == "__main__":
    main()
