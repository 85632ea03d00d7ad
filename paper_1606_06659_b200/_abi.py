"""ctypes mirror of include/countmc_b200.h and the product library loader.

The shared library is built in-tree (``paper_1606_06659_b200/lib``) by
``__graft_entry__.build()``.  Loading fails loudly when it is missing: there
is no CPU fallback for the sweep.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, c_char, c_double, c_int, c_long, c_longlong,
                    c_uint64, c_void_p)

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CMC_LIB_OVERRIDE") or os.path.join(HERE, "lib", "libcountmc_b200.so")

CMC_OK = 0
CMC_ERR_CONFIG = 1
CMC_ERR_STALL = 2
CMC_ERR_CUDA = 3
CMC_ERR_NCCL = 4
CMC_ERR_ARG = 5
CMC_ERR_LOAD = 6

CMC_PHASES = 6  # eps, gene (+ fused leaf sums), xi, hyper_a (or leaf_a), leaf_b, gene_contrast
PHASE_NAMES = ("eps", "gene", "xi", "hyper_a", "leaf_b", "gene_contrast")

CMC_SLICE_FAITHFUL = 0
CMC_CONJUGATE_DIRECT = 1

FAMILIES = {"beta_col": 0, "gamma": 1, "theta": 2, "sigma": 3, "nu": 4, "tau": 5}

# Exported symbols, one per C-ABI entry point in include/countmc_b200.h.
EXPORTS = [
    "cmc_version", "cmc_engine_create", "cmc_engine_destroy", "cmc_engine_dims",
    "cmc_engine_saved_genes", "cmc_engine_config", "cmc_engine_initial_state",
    "cmc_engine_set_state", "cmc_engine_get_state", "cmc_engine_iterate",
    "cmc_engine_run", "cmc_engine_begin", "cmc_engine_sweeps", "cmc_engine_sync",
    "cmc_engine_prepare", "cmc_engine_set_step_timing",
    "cmc_engine_stream", "cmc_engine_launches_per_sweep", "cmc_engine_profile",
    "cmc_engine_profile_phases",
    "cmc_engine_trace", "cmc_engine_diagnostics", "cmc_engine_write_results",
    "cmc_engine_get_output",
    "cmc_simulate", "cmc_engine_shard", "cmc_nccl_unique_id", "cmc_shard_bounds",
    "cmc_loopback_create", "cmc_loopback_destroy", "cmc_engine_shard_loopback",
    "cmc_engine_set_output",
    "cmc_counts_load", "cmc_counts_dims", "cmc_counts_data", "cmc_counts_gene",
    "cmc_counts_sample", "cmc_counts_labels", "cmc_counts_free", "cmc_estimate_offsets",
    "cmc_model_matrix_load", "cmc_offsets_load", "cmc_table_dims", "cmc_table_data",
    "cmc_table_name", "cmc_table_free",
]


class CmcError(ctypes.Structure):
    _fields_ = [("code", c_int), ("step", c_char * 16), ("index1", c_long),
                ("index2", c_long), ("iteration", c_long), ("x0", c_double),
                ("width", c_double), ("msg", c_char * 256)]


class CmcProblem(ctypes.Structure):
    _fields_ = [("G", c_long), ("N", c_long), ("L", c_long),
                ("counts", POINTER(c_longlong)), ("X", POINTER(c_double)),
                ("h", POINTER(c_double)), ("a", c_double), ("b", c_double),
                ("d", c_double), ("c", POINTER(c_double)), ("s", POINTER(c_double)),
                ("beta_prior", POINTER(c_int)), ("t_df", c_double)]


PRIORS = {"normal": 0, "laplace": 1, "t": 2, "horseshoe": 3}


class CmcRunConfig(ctypes.Structure):
    _fields_ = [("chains", c_long), ("iterations", c_long), ("burnin", c_long),
                ("tune_cutoff", c_long), ("thin", c_long), ("seed", c_uint64),
                ("max_step_out", c_int), ("max_shrink", c_int), ("w_init", c_double),
                ("save_genes", c_long), ("workers", c_int), ("sampler_mode", c_int),
                ("concurrent_chains", c_int)]


class CmcContrastSet(ctypes.Structure):
    _fields_ = [("n_contrasts", c_int), ("n_terms", POINTER(c_int)),
                ("n_coefs", POINTER(c_int)), ("threshold", POINTER(c_double)),
                ("family", POINTER(c_int)), ("index", POINTER(c_int)),
                ("coef", POINTER(c_double))]


class CmcDiagView(ctypes.Structure):
    _fields_ = [("rhat", POINTER(c_double)), ("mean", POINTER(c_double)),
                ("sd", POINTER(c_double)), ("ci_lo", POINTER(c_double)),
                ("ci_hi", POINTER(c_double)), ("flags", POINTER(c_int)),
                ("ess", POINTER(c_double)), ("ess_status", POINTER(c_int))]


class CmcOutputView(ctypes.Structure):
    _fields_ = [("acc_count", POINTER(c_long)), ("acc_mean", POINTER(c_double)),
                ("acc_meansq", POINTER(c_double)), ("acc_mean_c", POINTER(c_double)),
                ("acc_meansq_c", POINTER(c_double)),
                ("contrast_prob", POINTER(c_double)),
                ("contrast_count", POINTER(c_long)), ("samples", POINTER(c_double)),
                ("sample_iters", POINTER(c_long)), ("clamp_events", POINTER(c_uint64)),
                ("final_state", POINTER(c_double)), ("step_seconds", POINTER(c_double))]


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(POINTER(c_double))


def lptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(POINTER(c_long))


def iptr(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(POINTER(c_int))


class ProblemArrays:
    """Owns the numpy buffers a CmcProblem points into."""

    def __init__(self, counts, X, h, a, b, d, c, s, beta_prior=None, t_df=1.0):
        self.counts = np.ascontiguousarray(counts, dtype=np.int64)
        self.X = np.ascontiguousarray(X, dtype=np.float64)
        self.h = np.ascontiguousarray(h, dtype=np.float64)
        self.c = np.ascontiguousarray(c, dtype=np.float64)
        self.s = np.ascontiguousarray(s, dtype=np.float64)
        G, N = self.counts.shape
        L = self.X.shape[1]
        self.prior = None
        if beta_prior is not None and len(beta_prior):
            codes = [PRIORS[x] if isinstance(x, str) else int(x) for x in beta_prior]
            if len(codes) == 1 and L > 1:
                codes = codes * L
            self.prior = np.ascontiguousarray(codes, dtype=np.int32)
        self.xi = self.prior is not None and bool((self.prior != 0).any())
        self.struct = CmcProblem(G, N, L,
                                 self.counts.ctypes.data_as(POINTER(c_longlong)),
                                 dptr(self.X), dptr(self.h), float(a), float(b),
                                 float(d), dptr(self.c), dptr(self.s),
                                 self.prior.ctypes.data_as(POINTER(c_int))
                                 if self.prior is not None else None, float(t_df))


class ContrastArrays:
    """Flattens [(terms: [( [(family, index, coef)], threshold )])] into a
    CmcContrastSet (streaming.hpp ContrastSpec list)."""

    def __init__(self, contrasts):
        n_terms, n_coefs, thr, fam, idx, coef = [], [], [], [], [], []
        for terms in contrasts:
            n_terms.append(len(terms))
            for coefs, threshold in terms:
                n_coefs.append(len(coefs))
                thr.append(threshold)
                for f, i, cf in coefs:
                    fam.append(FAMILIES[f] if isinstance(f, str) else int(f))
                    idx.append(int(i))
                    coef.append(float(cf))
        self.n_terms = np.array(n_terms or [0], dtype=np.int32)
        self.n_coefs = np.array(n_coefs or [0], dtype=np.int32)
        self.thr = np.array(thr or [0.0], dtype=np.float64)
        self.fam = np.array(fam or [0], dtype=np.int32)
        self.idx = np.array(idx or [0], dtype=np.int32)
        self.coef = np.array(coef or [0.0], dtype=np.float64)
        self.struct = CmcContrastSet(len(contrasts), iptr(self.n_terms),
                                     iptr(self.n_coefs), dptr(self.thr),
                                     iptr(self.fam), iptr(self.idx), dptr(self.coef))


def make_config(chains=4, iterations=4000, burnin=2000, tune_cutoff=-1, thin=20,
                seed=1, max_step_out=100, max_shrink=1000, w_init=1.0,
                save_genes=20, workers=1, sampler_mode=CMC_SLICE_FAITHFUL,
                concurrent_chains=False) -> CmcRunConfig:
    return CmcRunConfig(chains, iterations, burnin, tune_cutoff, thin, seed,
                        max_step_out, max_shrink, w_init, save_genes, workers,
                        sampler_mode, int(bool(concurrent_chains)))


def sizes(G: int, N: int, L: int, xi: bool = False):
    """(S, T, A): packed state, tuning and accumulator lengths (xi: a ξ prior
    on some column adds a trailing G x L block to each)."""
    X = G * L if xi else 0
    S = G * N + G + G * L + 2 * L + 2 + X
    T = G * N + G + G * L + L + 2 + X
    A = 2 + 2 * L + G * L + G + G * N + X
    return S, T, A


_LIB = None


def load_library(path: str = LIB_PATH):
    """Load the CUDA product library; raises if it was not built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(
            f"countmc_b200 CUDA library missing at {path}; run "
            "`python -c 'import __graft_entry__ as g; g.build()'` first "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    E = POINTER(CmcError)
    lib.cmc_version.restype = ctypes.c_char_p
    lib.cmc_engine_create.argtypes = [POINTER(CmcProblem), POINTER(CmcRunConfig),
                                      POINTER(CmcContrastSet), c_int,
                                      POINTER(c_void_p), E]
    lib.cmc_engine_destroy.argtypes = [c_void_p]
    lib.cmc_engine_dims.argtypes = [c_void_p] + [POINTER(c_long)] * 7
    lib.cmc_engine_saved_genes.argtypes = [c_void_p, POINTER(c_long)]
    lib.cmc_engine_config.argtypes = [c_void_p, POINTER(CmcRunConfig)]
    lib.cmc_engine_initial_state.argtypes = [c_void_p, c_long, POINTER(c_double), E]
    lib.cmc_engine_set_state.argtypes = [c_void_p, c_long] + [POINTER(c_double)] * 3 + [E]
    lib.cmc_engine_get_state.argtypes = [c_void_p, c_long] + [POINTER(c_double)] * 3 + [E]
    lib.cmc_engine_iterate.argtypes = [c_void_p, c_long, c_long, POINTER(c_uint64), E]
    lib.cmc_engine_run.argtypes = [c_void_p, E]
    lib.cmc_engine_begin.argtypes = [c_void_p, E]
    lib.cmc_engine_sweeps.argtypes = [c_void_p, c_long, c_long, E]
    lib.cmc_engine_sync.argtypes = [c_void_p, E]
    lib.cmc_engine_prepare.argtypes = [c_void_p, c_long, E]
    lib.cmc_engine_set_step_timing.argtypes = [c_void_p, c_int]
    lib.cmc_engine_stream.argtypes = [c_void_p]
    lib.cmc_engine_stream.restype = c_void_p
    lib.cmc_engine_launches_per_sweep.argtypes = [c_void_p]
    lib.cmc_engine_profile.argtypes = [c_void_p, c_long, c_long, POINTER(c_double),
                                       POINTER(c_double), E]
    lib.cmc_engine_profile_phases.argtypes = [c_void_p, c_long, c_long, POINTER(c_double), E]
    lib.cmc_engine_trace.argtypes = [c_void_p, c_long, c_long, POINTER(ctypes.c_uint64), c_long,
                                     POINTER(c_long), E]
    lib.cmc_engine_diagnostics.argtypes = [c_void_p, POINTER(CmcDiagView), E]
    lib.cmc_engine_write_results.argtypes = [c_void_p, ctypes.c_char_p,
                                             POINTER(ctypes.c_char_p), POINTER(ctypes.c_char_p),
                                             c_double, E]
    lib.cmc_engine_get_output.argtypes = [c_void_p, c_long, POINTER(CmcOutputView), E]
    lib.cmc_simulate.argtypes = [c_long, c_long, c_long, POINTER(c_double),
                                 POINTER(c_double), c_double, c_double,
                                 POINTER(c_double), POINTER(c_double), c_uint64,
                                 POINTER(c_longlong), E]
    lib.cmc_engine_shard.argtypes = [c_void_p, c_int, c_int, c_void_p, E]
    lib.cmc_nccl_unique_id.argtypes = [c_void_p, E]
    lib.cmc_shard_bounds.argtypes = [c_long, c_int, c_int, POINTER(c_long), POINTER(c_long)]
    lib.cmc_loopback_create.argtypes = [c_int, POINTER(c_void_p), E]
    lib.cmc_loopback_destroy.argtypes = [c_void_p]
    lib.cmc_engine_shard_loopback.argtypes = [c_void_p, c_int, c_void_p, E]
    lib.cmc_engine_set_output.argtypes = [c_void_p, c_long, POINTER(CmcOutputView), E]
    lib.cmc_counts_load.argtypes = [ctypes.c_char_p, POINTER(c_void_p), E]
    lib.cmc_counts_dims.argtypes = [c_void_p, POINTER(c_long), POINTER(c_long), POINTER(c_int)]
    lib.cmc_counts_data.argtypes = [c_void_p]
    lib.cmc_counts_data.restype = POINTER(c_longlong)
    lib.cmc_counts_gene.argtypes = [c_void_p, c_long]
    lib.cmc_counts_gene.restype = ctypes.c_char_p
    lib.cmc_counts_sample.argtypes = [c_void_p, c_long]
    lib.cmc_counts_sample.restype = ctypes.c_char_p
    lib.cmc_counts_labels.argtypes = [c_void_p, c_int, POINTER(ctypes.c_char_p),
                                      POINTER(ctypes.c_size_t)]
    lib.cmc_counts_free.argtypes = [c_void_p]
    lib.cmc_counts_free.restype = None
    lib.cmc_model_matrix_load.argtypes = [ctypes.c_char_p, POINTER(c_void_p), E]
    lib.cmc_offsets_load.argtypes = [ctypes.c_char_p, POINTER(c_void_p), E]
    lib.cmc_table_dims.argtypes = [c_void_p, POINTER(c_long), POINTER(c_long)]
    lib.cmc_table_data.argtypes = [c_void_p]
    lib.cmc_table_data.restype = POINTER(c_double)
    lib.cmc_table_name.argtypes = [c_void_p, c_long]
    lib.cmc_table_name.restype = ctypes.c_char_p
    lib.cmc_table_free.argtypes = [c_void_p]
    lib.cmc_table_free.restype = None
    lib.cmc_estimate_offsets.argtypes = [c_long, c_long, POINTER(c_longlong),
                                         POINTER(c_double), E]
    _LIB = lib
    return lib
