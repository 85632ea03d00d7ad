#!/usr/bin/env python
"""Benchmark: MCMC gene-iterations/sec of the B200 Gibbs sweep.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step is one monitored Gibbs sweep (iterate + run_chain's Welford monitors,
per-gene heterosis contrast and thinning, P:src/engine.cpp:409-447) of every
chain.  The default workload is BASELINE.json configs[1]: Paschold-shaped
synthetic data, G = 39,656 genes per GPU, N = 16 samples, L = 5
(heterosis16x5), Normal beta prior, 4 chains (the reference RunConfig
default), widths tuned by 200 burn-in sweeps before timing.  Under torchrun
(N > 1) genes are sharded across ranks (weak scaling: 39,656 genes per GPU)
with an NCCL all-gather of the leaf partial sums per sweep.

--impl reference times the UNMODIFIED reference CPU sampler (compiled from
/root/reference into oracle/_ref) on all host threads on the same workload.
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

G_PER_GPU = 39656
N_SAMPLES = 16
THETA = [2.5, 0.2, 0.2, 0.0, 0.1]
SIGMA = [0.4, 0.25, 0.25, 0.15, 0.2]
PAPER_K20 = 2.27e6  # fbseqCUDA on a K20, PAPER.md:371 (different code, context only)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--chains", type=int, default=4)
    ap.add_argument("--genes-per-gpu", type=int, default=G_PER_GPU)
    ap.add_argument("--burnin", type=int, default=200)
    ap.add_argument("--e2e-burnin", type=int, default=2000)      # reference RunConfig default
    ap.add_argument("--e2e-iterations", type=int, default=4000)  # reference RunConfig default
    ap.add_argument("--e2e-reps", type=int, default=2)  # complete runs; the fastest is reported
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-xi", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    return ap.parse_args()


def problem(G, N=N_SAMPLES):
    from paper_1606_06659_b200 import SimSpec, builtin_design, generate
    X = builtin_design("heterosis16x5", N)
    counts = generate(SimSpec(G=G, N=N, X=X, nu=8.0, tau=0.7, theta=THETA,
                              sigma=SIGMA, seed=1)).counts
    return counts, X, np.zeros(N)


def bytes_per_gene_iter(N, L, n_gene_contrasts):
    """Minimum HBM bytes of one monitored gene-iteration:
    reads y 4N, eps 8N, w_eps 8N, gamma 8, w_gamma 8, beta 8L, w_beta 8L;
    writes eps 8N, gamma 8, beta 8L; compensated-Welford monitors (4 doubles
    read + written) for N+L+1 scalars; 16 B per per-gene contrast."""
    return 92 * N + 88 * L + 88 + 16 * n_gene_contrasts


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


def reference_rate(counts, X, h, burnin, warmup, steps=None, seconds=None, workers=None):
    """The reference's own iterate + monitors on all host threads, or on
    `workers` threads after an all-thread burn-in (oracle/_ref shim
    ref_bench_split).  Returns (gene-iter/s, threads, sweeps, s, kind)."""
    import oracle
    from paper_1606_06659_b200 import _abi
    all_threads = nproc()
    threads = workers or all_threads
    cfg = _abi.make_config(chains=1, burnin=burnin, iterations=10 ** 6, thin=20, seed=7,
                           save_genes=20, workers=threads)
    heter = [([("beta_col", 1, 2.0), ("beta_col", 3, 1.0)], 0.0),
             ([("beta_col", 2, 2.0), ("beta_col", 3, 1.0)], 0.0)]
    if oracle.ref_available():
        eng = oracle.RefEngine(counts, X, h, cfg, contrasts=[heter], workers=threads)
        kind = "reference"
    else:  # pragma: no cover - the built reference travels with the repo
        raise RuntimeError("oracle/_ref/libcountmc_ref.so missing")
    G = counts.shape[0]
    if steps is None:
        probe = eng.bench(threads, burnin + warmup, 3, burn_workers=all_threads)
        steps = max(3, int(seconds / max(probe / 3, 1e-6)))
    secs = eng.bench(threads, burnin + warmup, steps, burn_workers=all_threads)
    return G * steps / secs, threads, steps, secs, kind


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
    if rank != 0:
        return
    G = a.genes_per_gpu * world
    counts, X, h = problem(G)
    # --warmup W untimed sweeps after burn-in, then exactly --steps K timed sweeps
    rate, threads, steps, secs, kind = reference_rate(counts, X, h, a.burnin, a.warmup,
                                                      steps=a.steps)
    line = {
        "impl": "reference", "metric": "MCMC gene-iterations/sec", "value": rate,
        "unit": "gene-iter/s", "n_gpus": world, "steps": steps, "warmup": a.warmup,
        "ms_per_step": secs / steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic Paschold-shaped counts (heterosis16x5 design, seed 1)",
        "config": {"workload": f"paschold_G{G}_N16_L5_heterosis16x5", "G": G, "N": 16,
                   "L": 5, "chains": 1, "burnin": a.burnin, "contrasts": 1,
                   "sampler": "slice_faithful", "threads": threads},
        "cpu_baseline": {"value": rate, "unit": "gene-iter/s", "cores": threads, "kind": kind,
                         "sample": f"{steps} monitored sweeps of 1 chain at G={G} after "
                                   f"{a.burnin + a.warmup} burn-in sweeps, workers={threads}, "
                                   f"{cpu_model()}"},
        "e2e": {"value": rate, "unit": "gene-iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(a, rank, world, local_rank):
    import torch
    import paper_1606_06659_b200 as pkg
    from paper_1606_06659_b200 import (CountMatrix, GibbsEngine, ModelSpec, RunConfig,
                                       heterosis_contrast)
    from paper_1606_06659_b200._abi import CmcError
    dist = world > 1
    torch.cuda.set_device(local_rank)
    G = a.genes_per_gpu * world
    counts, X, h = problem(G)
    C, B, W, K = a.chains, a.burnin, a.warmup, a.steps
    prof_reps = 5
    # iterations cover warm-up, the clock probe (below), the timed steps and
    # the profile reps; monitors run on all of them like run_chain's
    cfg = RunConfig(chains=C, burnin=B, iterations=W + 20000 + K + prof_reps, thin=20, seed=7,
                    save_genes=20)
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg,
                      contrasts=[heterosis_contrast()], device=local_rank)
    if dist:
        import torch.distributed as td
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(GibbsEngine.nccl_unique_id()), dtype=torch.uint8))
        td.broadcast(uid, 0)
        eng.shard(rank, world, bytes(uid.cpu().numpy().tobytes()))
    lib, hd, err = eng._lib, eng.handle, CmcError()

    def ok(rc):
        if rc:
            raise RuntimeError(err.msg.decode())

    ok(lib.cmc_engine_begin(hd, byref(err)))
    stream = torch.cuda.ExternalStream(lib.cmc_engine_stream(hd))
    # burn-in (tuning active, no monitors), timed separately:
    # sweeps 1..5 start from w_init = 1 (the divergent-slice-loop proxy,
    # config 3); the next 50 include the one-time capture of the sweep graph;
    # the rest is the steady burn-in rate
    nb0 = min(5, B)
    nb1 = min(50, B - nb0)
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
    burnin = {"value": C * G * n_rest / (burn_rest_ms * 1e-3) if n_rest else None,
              "unit": "gene-iter/s", "sweeps": B,
              "ms_per_sweep": burn_rest_ms / n_rest if n_rest else None,
              "first_sweeps": nb0, "first_ms_per_sweep": burn_first_ms / max(nb0, 1),
              "graph_capture_chunk_ms": burn_cap_ms,
              "note": "burn-in sweeps (tuning on, no monitors), one GPU, device-timed: value and "
                      "ms_per_sweep over sweeps 56..B; first_* are sweeps 1..5 from w_init=1 "
                      "(wide, divergent slice loops); graph_capture_chunk_ms is sweeps 6..55 "
                      "including the one-time CUDA-graph capture"}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    # clocks are sampled under load: untimed monitored sweeps keep the GPU busy
    # for ~0.4 s right before the timed region, inside the sampler's window
    n_probe = min(20000, int(400.0 / max(warm_ms, 1e-3)))
    m0 = B + 1 + W + n_probe
    clocks = Clocks(local_rank)
    clocks.start()
    time.sleep(0.1)  # nvidia-smi start-up
    ok(lib.cmc_engine_sweeps(hd, B + 1 + W, m0, byref(err)))
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
    value = C * G * K / (ms * 1e-3)
    # per-sweep kernels of every lane + one iteration-advance kernel per 50-sweep graph
    launches = K * lib.cmc_engine_launches_per_sweep(hd) + (K // 50) + (1 if K % 50 else 0)

    # dominant kernel timed live with events on the engine stream
    gene_ms, tail_ms = c_double(), c_double()
    roofline = None
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    if not dist:
        ok(lib.cmc_engine_profile(hd, m0 + K, prof_reps, byref(gene_ms), byref(tail_ms),
                                  byref(err)))
        bpg = bytes_per_gene_iter(N_SAMPLES, 5, 1)
        per_launch = C * G * bpg
        achieved = per_launch / (gene_ms.value * 1e-3) / 1e9
        peak = peaks.get("hbm_gbs", 6650.0)
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "gene_sweep_traffic.json")
        if os.path.exists(tpath):
            tj = json.load(open(tpath))
            if tj.get("chains") == C and tj.get("G") == G:
                traffic = tj.get("dram_bytes_per_launch")
        # the bound the sweep actually sits on: warp-instruction issue
        # (profiles/sweep_instructions.json: ncu count per 4-chain sweep)
        issue = None
        ipath = os.path.join(ROOT, "profiles", "sweep_instructions.json")
        if os.path.exists(ipath):
            ij = json.load(open(ipath))
            if ij.get("chains") == C and ij.get("G") == G:
                mhz = (clk or {}).get("sm_mhz") or 1965.0
                ipeak = 148 * 4 * mhz * 1e6          # 1 warp-instruction / scheduler / clock
                iach = ij["warp_inst_per_sweep"] / (ms / K * 1e-3)
                issue = {"bound": "issue", "achieved": iach, "peak": ipeak,
                         "unit": "warp-inst/s", "frac": iach / ipeak,
                         "warp_inst_per_sweep": ij["warp_inst_per_sweep"],
                         "note": "ncu instruction count of eps+gene+leaf kernels per 4-chain "
                                 "sweep over the live ms_per_step; peak = 148 SMs x 4 "
                                 "schedulers x SM clock"}
        roofline = {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "kernel": "eps_sweep_kernel + gene_sweep_kernel (the fused sweep; timed together)",
            "algorithmic_bytes_per_launch": per_launch,
            "bytes_per_gene_iter": bpg,
            "kernel_ms": gene_ms.value, "tail_ms": tail_ms.value,
            "kernel_share_of_step": gene_ms.value / (gene_ms.value + tail_ms.value),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s",
            "note": "the sweep is issue/latency bound, not HBM bound (see issue_roofline "
                    "and DESIGN.md 'Roofline': measured FP64 36.3 TFLOP/s DFMA, 8.1e11 exp/s, "
                    "Philox 1.1e11 blocks/s)",
            "issue_roofline": issue,
        }
    del eng
    torch.cuda.synchronize()

    # BASELINE configs[1] names Laplace priors, configs[2] t and horseshoe:
    # the xi extension (not in the reference; parity unpinned)
    # timed the same way on the same data.  The headline stays the normal
    # prior, the only model the reference (and so the reference arm) has.
    xi_rates = None
    if not dist and not a.no_xi:
        xi_rates = {}
        from paper_1606_06659_b200 import PriorConfig
        for name in ("laplace", "t", "horseshoe"):
            spec = ModelSpec(X, h, PriorConfig(beta_prior=[name], t_df=3.0))
            ex = GibbsEngine(CountMatrix(counts), spec,
                             RunConfig(chains=C, burnin=B, iterations=W + K, thin=20, seed=7,
                                       save_genes=20),
                             contrasts=[heterosis_contrast()], device=local_rank)
            lx, hx = ex._lib, ex.handle
            ok(lx.cmc_engine_begin(hx, byref(err)))
            ok(lx.cmc_engine_sweeps(hx, 1, B + 1 + W, byref(err)))
            ok(lx.cmc_engine_sync(hx, byref(err)))
            sx = torch.cuda.ExternalStream(lx.cmc_engine_stream(hx))
            x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            x0.record(sx)
            ok(lx.cmc_engine_sweeps(hx, B + 1 + W, B + 1 + W + K, byref(err)))
            x1.record(sx)
            ok(lx.cmc_engine_sync(hx, byref(err)))
            torch.cuda.synchronize()
            xms = x0.elapsed_time(x1)
            xi_rates[name] = {"value": C * G * K / (xms * 1e-3), "ms_per_step": xms / K}
            del ex
        xi_rates["note"] = ("beta_gl ~ N(theta_l, sigma_l^2 xi_gl) with a xi slice step per "
                            "(gene, column); t with k = 3; same data, chains, burn-in and "
                            "device timing as value; extension, not in the reference")

    # BASELINE configs 4 and 5 on this GPU (parity cases, not the headline):
    # same chains and device timing, 100 burn-in sweeps, 20 timed
    other = None
    if not dist and not a.no_other_configs:
        other = {}
        for name, Gx, Nx in (("G1000000_N16", 1_000_000, 16), ("G200000_N64", 200_000, 64)):
            cx, Xx, hx_ = problem(Gx, Nx)
            ex = GibbsEngine(CountMatrix(cx), ModelSpec(Xx, hx_),
                             RunConfig(chains=C, burnin=100, iterations=40, thin=20, seed=7,
                                       save_genes=20),
                             contrasts=[heterosis_contrast()], device=local_rank)
            lx, hdx = ex._lib, ex.handle
            ok(lx.cmc_engine_begin(hdx, byref(err)))
            ok(lx.cmc_engine_sweeps(hdx, 1, 106, byref(err)))
            ok(lx.cmc_engine_sync(hdx, byref(err)))
            sx = torch.cuda.ExternalStream(lx.cmc_engine_stream(hdx))
            y0, y1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            y0.record(sx)
            ok(lx.cmc_engine_sweeps(hdx, 106, 126, byref(err)))
            y1.record(sx)
            ok(lx.cmc_engine_sync(hdx, byref(err)))
            torch.cuda.synchronize()
            yms = y0.elapsed_time(y1) / 20
            other[name] = {"value": C * Gx / (yms * 1e-3), "ms_per_step": yms, "chains": C}
            del ex, cx
        other["note"] = ("BASELINE configs 4 (G=1M, N=16; one GPU) and 5 (G=200k, N=64), "
                         "heterosis16x5, normal prior, 100 burn-in then 20 device-timed "
                         "monitored sweeps")

    # end to end through the public API from host arrays: create (H2D of
    # counts + initial states), run() (burn-in + iterations), all outputs D2H
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
            uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                uid.copy_(torch.frombuffer(bytearray(GibbsEngine.nccl_unique_id()),
                                           dtype=torch.uint8))
            torch.distributed.broadcast(uid, 0)
            eng2.shard(rank, world, bytes(uid.cpu().numpy().tobytes()))
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
    S, T, A = pkg.sizes(G, N_SAMPLES, 5)
    h2d = counts.size * 8 + X.size * 8 + h.size * 8 + C * (S + 2 * T) * 8
    d2h = C * (4 * A * 8 + S * 8 + G * 8 + outs[0].samples.size * 8)
    e2e = {"value": C * G * (BE + E) / wall, "unit": "gene-iter/s",
           "h2d_bytes_per_step": h2d / (BE + E), "d2h_bytes_per_step": d2h / (BE + E),
           "wall_s": wall, "wall_s_all": walls, "sweeps": BE + E, "burnin": BE,
           "iterations": E,
           "post_burnin_only_value": C * G * E / wall,
           "note": "one GibbsEngine(...).run() with the reference's default RunConfig "
                   "(chains 4, burnin 2000, iterations 4000), host wall clock: host count "
                   "matrix in (H2D), every sweep, all ChainOutputs out (D2H).  An MCMC run "
                   "has one input (the counts) and one result (the ChainOutputs), so the "
                   "per-step byte figures are those run totals over the sweeps; a per-sweep "
                   "host round trip would only serialise the pipeline.  value counts every "
                   "sweep the call ran (burn-in sweeps are gene-iterations too, and cost "
                   "slightly more: tuning); post_burnin_only_value charges the whole wall "
                   "time to the 4000 monitored sweeps; the fastest of e2e_reps complete "
                   "runs (wall_s_all lists each; max over ranks per run)"}

    if rank != 0:
        return
    cpu = None
    if not a.no_cpu_baseline and world == 1:
        try:
            rate, threads, steps, secs, kind = reference_rate(counts, X, h, B, W,
                                                              seconds=a.cpu_seconds)
            cpu = {"value": rate, "unit": "gene-iter/s", "cores": threads, "kind": kind,
                   "sample": f"{steps} monitored sweeps of 1 chain at G={G} after {B + W} "
                             f"burn-in sweeps, reference iterate()+monitors, workers={threads}, "
                             f"{cpu_model()}"}
            r1, _, s1, _, _ = reference_rate(counts, X, h, B, W, seconds=a.cpu_seconds / 3,
                                             workers=1)
            cpu["single_core"] = {"value": r1, "cores": 1,
                                  "sample": f"{s1} monitored sweeps, workers=1 (burn-in on "
                                            f"all threads)"}
        except Exception as ex:  # report, never fake
            cpu = {"value": None, "unit": "gene-iter/s", "cores": nproc(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}
    line = {
        "metric": "MCMC gene-iterations/sec", "value": value, "unit": "gene-iter/s",
        "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms / K,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic Paschold-shaped counts (heterosis16x5 design, seed 1), "
                "random-initialised chains",
        "config": {"workload": f"paschold_G{G}_N16_L5_heterosis16x5", "G": G,
                   "G_per_gpu": a.genes_per_gpu, "N": 16, "L": 5, "chains": C,
                   "burnin": B, "thin": 20, "contrasts": "heterosis (per gene)",
                   "sampler": "slice_faithful", "prior": "normal (reference has no Laplace)",
                   "parallelism": f"gene-shard x{world}" if dist else "single GPU",
                   "l2": "inputs larger than L2: ~%.0f MB touched per sweep vs 126 MB L2"
                         % (C * G * bytes_per_gene_iter(16, 5, 1) / 1e6 + G * 16 * 8 / 1e6)},
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
    if world > 1:
        import torch
        import torch.distributed as td
        torch.cuda.set_device(local_rank)
        td.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_b200(a, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as td
            td.destroy_process_group()


if __name__ == "__main__":
    main()
