"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes harness over

* ``oracle/liboracle.so`` — the plain-C restatement of the reference sweep
  (``countmc_oracle.c``), and
* ``oracle/_ref/libcountmc_ref.so`` — the unmodified reference library
  compiled from /root/reference by ``oracle/Makefile`` (travels to the GPU
  box as a built file; the reference sources do not).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this package.  The product (``paper_1606_06659_b200``) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, byref, c_double, c_int, c_long, c_longlong, c_uint64, c_void_p

import numpy as np

from paper_1606_06659_b200 import _abi
from paper_1606_06659_b200._abi import (CmcError, CmcOutputView, ContrastArrays,
                                        ProblemArrays, dptr, lptr, sizes)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcountmc_ref.so")
REF_SRC = "/root/reference/proj"

_ORC = None
_REF = None


def build(ref: bool = True):
    """Compile the oracle (and, when the reference sources exist, oracle/_ref)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def load_oracle():
    global _ORC
    if _ORC is not None:
        return _ORC
    if not os.path.exists(ORACLE_SO):
        build(ref=False)
    lib = ctypes.CDLL(ORACLE_SO)
    E = POINTER(CmcError)
    D = POINTER(c_double)
    U = POINTER(c_uint64)
    lib.orc_philox4x64.argtypes = [U, U, U]
    lib.orc_normal_quantile.argtypes = [c_double]
    lib.orc_normal_quantile.restype = c_double
    lib.orc_stream_u01.argtypes = [c_uint64] * 4 + [c_long, D]
    lib.orc_clamped_exp.argtypes = [c_double, U]
    lib.orc_clamped_exp.restype = c_double
    lib.orc_log_fc_epsilon.argtypes = [c_longlong, c_double, c_double, c_double, c_double, U]
    lib.orc_log_fc_epsilon.restype = c_double
    lib.orc_gamma_fc_params.argtypes = [c_double, c_double, D, c_long, D, D]
    lib.orc_log_invgamma.argtypes = [c_double] * 3
    lib.orc_log_invgamma.restype = c_double
    lib.orc_log_gamma_rate.argtypes = [c_double] * 3
    lib.orc_log_gamma_rate.restype = c_double
    lib.orc_log_fc_nu.argtypes = [c_double, c_long, c_double, c_double, c_double, c_double]
    lib.orc_log_fc_nu.restype = c_double
    lib.orc_tau_fc_params.argtypes = [c_double, c_double, c_long, c_double, c_double, D, D]
    lib.orc_theta_fc_params.argtypes = [c_double, c_long, c_double, c_double, D, D]
    lib.orc_log_fc_sigma.argtypes = [c_double, c_long, c_double, c_double]
    lib.orc_log_fc_sigma.restype = c_double
    lib.orc_tune_update.argtypes = [D, D, c_long, c_double, c_void_p]
    lib.orc_slice_chain.argtypes = [c_int, c_double, c_long, c_long, c_double, c_uint64, D]
    lib.orc_log_fc_xi.argtypes = [c_int, c_double, c_double, c_double]
    lib.orc_log_fc_xi.restype = c_double
    lib.orc_pairwise_sum.argtypes = [D, ctypes.c_size_t]
    lib.orc_pairwise_sum.restype = c_double
    lib.orc_det_sum.argtypes = [D, c_long]
    lib.orc_det_sum.restype = c_double
    lib.orc_moments_stream.argtypes = [D, c_long, D, D]
    lib.orc_disjunction_combine.argtypes = [c_double] * 3
    lib.orc_disjunction_combine.restype = c_double
    lib.orc_engine_create.argtypes = [POINTER(_abi.CmcProblem), POINTER(_abi.CmcRunConfig),
                                      POINTER(_abi.CmcContrastSet), POINTER(c_void_p), E]
    lib.orc_engine_destroy.argtypes = [c_void_p]
    lib.orc_engine_config.argtypes = [c_void_p, POINTER(_abi.CmcRunConfig)]
    lib.orc_engine_n_saved.argtypes = [c_void_p]
    lib.orc_engine_n_saved.restype = c_long
    lib.orc_engine_saved_genes.argtypes = [c_void_p, POINTER(c_long)]
    lib.orc_initial_state.argtypes = [c_void_p, c_long, D]
    lib.orc_iterate.argtypes = [c_void_p, D, D, D, c_long, c_long, U, E]
    lib.orc_run_chain.argtypes = [c_void_p, c_long, POINTER(CmcOutputView), E]
    _ORC = lib
    return lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def load_ref():
    global _REF
    if _REF is not None:
        return _REF
    if not os.path.exists(REF_SO):
        raise RuntimeError(f"reference library not built at {REF_SO}")
    lib = ctypes.CDLL(REF_SO)
    E = POINTER(CmcError)
    D = POINTER(c_double)
    U = POINTER(c_uint64)
    lib.ref_engine_create.argtypes = [POINTER(_abi.CmcProblem), POINTER(_abi.CmcRunConfig),
                                      POINTER(_abi.CmcContrastSet), POINTER(c_void_p), E]
    lib.ref_engine_destroy.argtypes = [c_void_p]
    lib.ref_engine_n_saved.argtypes = [c_void_p]
    lib.ref_engine_n_saved.restype = c_long
    lib.ref_engine_saved_genes.argtypes = [c_void_p, POINTER(c_long)]
    lib.ref_engine_tune_cutoff.argtypes = [c_void_p]
    lib.ref_engine_tune_cutoff.restype = c_long
    lib.ref_initial_state.argtypes = [c_void_p, c_long, D]
    lib.ref_iterate.argtypes = [c_void_p, D, D, D, c_long, c_long, c_int, U, E]
    lib.ref_run.argtypes = [c_void_p, POINTER(CmcOutputView), E]
    lib.ref_bench.argtypes = [c_void_p, c_int, c_long, c_long]
    lib.ref_bench.restype = c_double
    lib.ref_write_results.argtypes = [c_void_p, ctypes.c_char_p, POINTER(ctypes.c_char_p),
                                      c_double, D, E]
    lib.ref_bench_split.argtypes = [c_void_p, c_int, c_int, c_long, c_long]
    lib.ref_bench_split.restype = c_double
    lib.ref_bench_chains.argtypes = [c_void_p, c_int, c_int, c_long, c_long, c_long]
    lib.ref_bench_chains.restype = c_double
    lib.ref_hardware_threads.restype = c_int
    I = POINTER(c_int)
    lib.ref_diagnostics.argtypes = [c_void_p, D, I, D, D, D, D, D, I, E]
    lib.ref_philox.argtypes = [U, U, U]
    lib.ref_normal_quantile.argtypes = [c_double]
    lib.ref_normal_quantile.restype = c_double
    lib.ref_stream_u01.argtypes = [c_uint64] * 4 + [c_long, D]
    lib.ref_stream_gamma.argtypes = [c_uint64, c_uint64, c_double, c_double, c_long, D]
    lib.ref_log_fc_epsilon.argtypes = [c_longlong] + [c_double] * 4
    lib.ref_log_fc_epsilon.restype = c_double
    lib.ref_log_fc_nu.argtypes = [c_double, c_long, c_double, c_double, c_double, c_double]
    lib.ref_log_fc_nu.restype = c_double
    lib.ref_log_fc_sigma.argtypes = [c_double, c_long, c_double, c_double]
    lib.ref_log_fc_sigma.restype = c_double
    lib.ref_pairwise_sum.argtypes = [D, c_long]
    lib.ref_pairwise_sum.restype = c_double
    lib.ref_load_counts.argtypes = [ctypes.c_char_p, POINTER(c_longlong), c_long,
                                    ctypes.c_char_p, c_long, POINTER(c_long), POINTER(c_long),
                                    I, ctypes.c_char_p]
    lib.ref_load_table.argtypes = [ctypes.c_char_p, c_int, D, c_long, POINTER(c_long),
                                   POINTER(c_long), ctypes.c_char_p]
    lib.ref_estimate_offsets.argtypes = [c_long, c_long, POINTER(c_longlong), D,
                                         ctypes.c_char_p]
    lib.ref_generate.argtypes = [c_long, c_long, c_long, D, D, c_double, c_double, D, D,
                                 c_uint64, POINTER(c_longlong), ctypes.c_char_p]
    lib.ref_builtin_design.argtypes = [c_long, D]
    _REF = lib
    return lib


class StallError(RuntimeError):
    def __init__(self, err: CmcError):
        super().__init__(err.msg.decode())
        self.step = err.step.decode()
        self.index1, self.index2 = err.index1, err.index2
        self.x0, self.width, self.iteration = err.x0, err.width, err.iteration


class ConfigErr(ValueError):
    pass


def _check(rc, err):
    if rc == 0:
        return
    if rc == _abi.CMC_ERR_STALL:
        raise StallError(err)
    if rc == _abi.CMC_ERR_CONFIG:
        raise ConfigErr(err.msg.decode())
    raise RuntimeError(err.msg.decode())


def new_outputs(G, N, L, n_saved, n_rows, n_prob, n_contrasts, xi=False):
    S, _, A = sizes(G, N, L, xi)
    ncols = 2 + 2 * L + n_saved * (L + 1)
    o = dict(count=np.zeros(1, np.int64), mean=np.zeros(A), meansq=np.zeros(A),
             mean_c=np.zeros(A), meansq_c=np.zeros(A), prob=np.zeros(max(1, n_prob)),
             ccount=np.zeros(max(1, n_contrasts), np.int64),
             samples=np.zeros(max(1, ncols * n_rows)), iters=np.zeros(max(1, n_rows), np.int64),
             clamps=np.zeros(1, np.uint64), final=np.zeros(S), secs=np.zeros(7))
    view = CmcOutputView(lptr(o["count"]), dptr(o["mean"]), dptr(o["meansq"]),
                         dptr(o["mean_c"]), dptr(o["meansq_c"]), dptr(o["prob"]),
                         lptr(o["ccount"]), dptr(o["samples"]), lptr(o["iters"]),
                         o["clamps"].ctypes.data_as(POINTER(c_uint64)), dptr(o["final"]),
                         dptr(o["secs"]))
    return o, view


class _Base:
    def __init__(self, counts, X, h, cfg: _abi.CmcRunConfig, contrasts=(), priors=None):
        G, N = counts.shape
        L = X.shape[1]
        pr = priors or {}
        self.G, self.N, self.L = G, N, L
        self.cfg = cfg
        self.prob = ProblemArrays(counts, X, h, pr.get("a", 1.0), pr.get("b", 1.0),
                                  pr.get("d", 1000.0), pr.get("c", [10.0] * L),
                                  pr.get("s", [100.0] * L), pr.get("beta_prior"),
                                  pr.get("t_df", 1.0))
        self.xi = self.prob.xi
        self.contrasts = list(contrasts)
        self.ctr = ContrastArrays(self.contrasts)


class OracleEngine(_Base):
    """The C restatement (countmc_oracle.c) behind a packed-array API."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.lib = load_oracle()
        err = CmcError()
        h = c_void_p()
        _check(self.lib.orc_engine_create(byref(self.prob.struct), byref(self.cfg),
                                          byref(self.ctr.struct) if self.contrasts else None,
                                          byref(h), byref(err)), err)
        self.h = h
        rc = _abi.CmcRunConfig()
        self.lib.orc_engine_config(h, byref(rc))
        self.resolved = rc

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_engine_destroy(self.h)

    def saved_genes(self):
        n = self.lib.orc_engine_n_saved(self.h)
        out = np.zeros(max(1, n), np.int64)
        self.lib.orc_engine_saved_genes(self.h, lptr(out))
        return out[:n]

    def initial_state(self, chain):
        S, _, _ = sizes(self.G, self.N, self.L, self.xi)
        st = np.zeros(S)
        self.lib.orc_initial_state(self.h, chain, dptr(st))
        return st

    def iterate(self, st, tw, ta, chain, m):
        err = CmcError()
        cl = c_uint64(0)
        rc = self.lib.orc_iterate(self.h, dptr(st), dptr(tw), dptr(ta), chain, m, byref(cl),
                                  byref(err))
        _check(rc, err)
        return cl.value

    def run_chain(self, chain):
        n_prob = sum(self.G if any(f in ("beta_col", "gamma", 0, 1) for t in c for f, _, _ in t[0])
                     else 1 for c in self.contrasts)
        n_rows = self.resolved.iterations // self.resolved.thin
        o, view = new_outputs(self.G, self.N, self.L, len(self.saved_genes()), n_rows, n_prob,
                              len(self.contrasts), self.xi)
        err = CmcError()
        _check(self.lib.orc_run_chain(self.h, chain, byref(view), byref(err)), err)
        return o


class RefEngine(_Base):
    """The compiled reference (oracle/_ref) behind the same packed API."""

    def __init__(self, *a, workers=1, **k):
        super().__init__(*a, **k)
        self.lib = load_ref()
        self.workers = workers
        err = CmcError()
        h = c_void_p()
        _check(self.lib.ref_engine_create(byref(self.prob.struct), byref(self.cfg),
                                          byref(self.ctr.struct) if self.contrasts else None,
                                          byref(h), byref(err)), err)
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_engine_destroy(self.h)

    def saved_genes(self):
        n = self.lib.ref_engine_n_saved(self.h)
        out = np.zeros(max(1, n), np.int64)
        self.lib.ref_engine_saved_genes(self.h, lptr(out))
        return out[:n]

    def initial_state(self, chain):
        S, _, _ = sizes(self.G, self.N, self.L)
        st = np.zeros(S)
        self.lib.ref_initial_state(self.h, chain, dptr(st))
        return st

    def iterate(self, st, tw, ta, chain, m):
        err = CmcError()
        cl = c_uint64(0)
        rc = self.lib.ref_iterate(self.h, dptr(st), dptr(tw), dptr(ta), chain, m,
                                  self.workers, byref(cl), byref(err))
        _check(rc, err)
        return cl.value

    def run(self):
        n_prob = sum(self.G if any(f in ("beta_col", "gamma", 0, 1) for t in c for f, _, _ in t[0])
                     else 1 for c in self.contrasts)
        n_rows = self.cfg.iterations // self.cfg.thin
        outs = [new_outputs(self.G, self.N, self.L, len(self.saved_genes()), n_rows, n_prob,
                            len(self.contrasts)) for _ in range(self.cfg.chains)]
        views = (CmcOutputView * self.cfg.chains)(*[v for _, v in outs])
        err = CmcError()
        _check(self.lib.ref_run(self.h, views, byref(err)), err)
        return [o for o, _ in outs]

    def diagnostics(self, n_cols):
        """Reference rows (rhat, flags, mean, sd, lo, hi) and per-column ESS."""
        G, L = self.G, self.L
        R = 2 + 2 * L + G * (L + 1)
        out = {k: np.zeros(R) for k in ("rhat", "mean", "sd", "lo", "hi")}
        out["flags"] = np.zeros(R, np.int32)
        out["ess"] = np.zeros(max(1, n_cols))
        out["ess_status"] = np.zeros(max(1, n_cols), np.int32)
        I = lambda a: a.ctypes.data_as(POINTER(c_int))
        err = CmcError()
        _check(self.lib.ref_diagnostics(self.h, dptr(out["rhat"]), I(out["flags"]),
                                        dptr(out["mean"]), dptr(out["sd"]), dptr(out["lo"]),
                                        dptr(out["hi"]), dptr(out["ess"]), I(out["ess_status"]),
                                        byref(err)), err)
        return out

    def write_results(self, outdir, genes=None, wall_seconds=0.0):
        """run() then the reference's write_results into outdir; returns the
        seconds write_results itself took."""
        gl = None
        if genes is not None:
            gl = (ctypes.c_char_p * len(genes))(*[g.encode() for g in genes])
        secs = c_double()
        err = CmcError()
        rc = self.lib.ref_write_results(self.h, str(outdir).encode(), gl, wall_seconds,
                                        ctypes.byref(secs), ctypes.byref(err))
        if rc == _abi.CMC_ERR_CONFIG:
            raise ConfigErr(err.msg.decode())
        if rc:
            raise StallError(err.msg.decode())
        return secs.value

    def bench(self, workers, burn, sweeps, burn_workers=None, chains=1):
        """Seconds of `chains` x `sweeps` monitored sweeps (chains in sequence,
        as run()), each chain after `burn` untimed burn-in sweeps."""
        return self.lib.ref_bench_chains(self.h, burn_workers or workers, workers, chains,
                                         burn, sweeps)


def heterosis16x5(N=16):
    A = np.array([[1, 1, -1, 0], [1, -1, 1, 0], [1, 1, 1, 1], [1, 1, 1, -1]], float)
    block = [1, 1, -1, -1]
    X = np.zeros((N, 5))
    for n in range(N):
        X[n, :4] = A[(n % 16) // 4]
        X[n, 4] = block[n % 4]
    return X


def ref_generate(G, N, nu, tau, theta, sigma, seed, X=None, h=None):
    """The reference's own synthetic data: generate() (P:src/simulate.cpp:
    28-90), with builtin_design("heterosis16x5", N) when X is None.
    Returns (counts G x N int64, X N x L)."""
    lib = load_ref()
    if X is None:
        L = len(theta)
        X = np.zeros((N, L))
        lib.ref_builtin_design(N, X.ctypes.data_as(POINTER(c_double)))
        Xp = None
    else:
        X = np.ascontiguousarray(X, dtype=np.float64)
        L = X.shape[1]
        Xp = X.ctypes.data_as(POINTER(c_double))
    th = np.ascontiguousarray(theta, dtype=np.float64)
    sg = np.ascontiguousarray(sigma, dtype=np.float64)
    hh = None if h is None else np.ascontiguousarray(h, dtype=np.float64)
    out = np.zeros((G, N), np.int64)
    msg = ctypes.create_string_buffer(256)
    rc = lib.ref_generate(G, N, L, Xp, None if hh is None else hh.ctypes.data_as(POINTER(c_double)),
                          nu, tau, th.ctypes.data_as(POINTER(c_double)),
                          sg.ctypes.data_as(POINTER(c_double)), seed,
                          out.ctypes.data_as(POINTER(c_longlong)), msg)
    if rc:
        raise ConfigErr(msg.value.decode(errors="replace"))
    return out, X


def ref_load_counts(path):
    """The reference's own load_counts (P:src/io.cpp:125-164).  Returns
    (counts, genes, samples, duplicate_genes) or raises RefLoadError /
    ConfigErr with the reference's message."""
    lib = load_ref()
    cap_cells, cap_names = 1 << 16, 1 << 20
    while True:
        cells = np.zeros(cap_cells, np.int64)
        names = ctypes.create_string_buffer(cap_names)
        G, N, dup = c_long(), c_long(), ctypes.c_int()
        msg = ctypes.create_string_buffer(256)
        rc = lib.ref_load_counts(str(path).encode(),
                                 cells.ctypes.data_as(POINTER(c_longlong)), cap_cells,
                                 names, cap_names, ctypes.byref(G), ctypes.byref(N),
                                 ctypes.byref(dup), msg)
        if rc == -1:
            cap_cells = max(cap_cells, G.value * N.value)
            cap_names *= 4
            continue
        if rc == 6:
            raise RefLoadError(msg.value.decode(errors="replace"))
        if rc == 1:
            raise ConfigErr(msg.value.decode(errors="replace"))
        G, N = G.value, N.value
        parts = names.raw.split(b"\0")[:N + G]
        samples = [p.decode(errors="surrogateescape") for p in parts[:N]]
        genes = [p.decode(errors="surrogateescape") for p in parts[N:]]
        return cells[:G * N].reshape(G, N).copy(), genes, samples, bool(dup.value)


def ref_load_table(path, which):
    """The reference's load_model_matrix (which=0) or load_offsets (1)."""
    lib = load_ref()
    cap = 1 << 16
    out = np.zeros(cap)
    r, c = c_long(), c_long()
    msg = ctypes.create_string_buffer(256)
    rc = lib.ref_load_table(str(path).encode(), which, out.ctypes.data_as(POINTER(c_double)),
                            cap, ctypes.byref(r), ctypes.byref(c), msg)
    if rc == 6:
        raise RefLoadError(msg.value.decode(errors="replace"))
    assert rc == 0
    return out[:r.value * c.value].reshape(r.value, c.value).copy()


def ref_estimate_offsets(counts):
    """The reference's estimate_offsets (P:src/model.cpp:21-68)."""
    lib = load_ref()
    y = np.ascontiguousarray(counts, dtype=np.int64)
    h = np.zeros(y.shape[1])
    msg = ctypes.create_string_buffer(256)
    rc = lib.ref_estimate_offsets(y.shape[0], y.shape[1], y.ctypes.data_as(POINTER(c_longlong)),
                                  h.ctypes.data_as(POINTER(c_double)), msg)
    if rc:
        raise ConfigErr(msg.value.decode(errors="replace"))
    return h


class RefLoadError(RuntimeError):
    """LoadError raised by the reference loader."""
