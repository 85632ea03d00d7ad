"""Host-side mirror of the reference countmc engine API over the C-ABI.

Names, argument meaning and error behaviour follow the reference headers
(P: = /root/reference/proj/):

* ``RunConfig`` / ``SliceConfig``    P:include/countmc/engine.hpp:21-36, slice.hpp:11-17
* ``ChainState``                     P:include/countmc/types.hpp:86-108
* ``TuningState``                    P:include/countmc/engine.hpp:58-74
* ``ChainOutput``                    P:include/countmc/engine.hpp:90-108
* ``GibbsEngine``                    P:include/countmc/engine.hpp:110-159
* ``ConfigError``/``SamplerStallError`` P:include/countmc/errors.hpp:10-71

Every sweep runs in the CUDA library (``lib/libcountmc_b200.so``); this
module only marshals arrays.  The library is required: nothing here computes
a sweep on the CPU.
"""
from __future__ import annotations

import ctypes
from ctypes import byref, c_long, c_uint64, c_void_p
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import (CmcError, CmcOutputView, ContrastArrays, ProblemArrays, dptr,
                   load_library, lptr, sizes)


class ConfigError(ValueError):
    """Bad configuration or inputs (reference ConfigError, exit code 1)."""


class SamplerStallError(RuntimeError):
    """Slice shrink loop exceeded max_shrink (reference SamplerStallError)."""

    def __init__(self, msg, step="", index1=-1, index2=-1, x0=0.0, width=0.0,
                 iteration=0):
        super().__init__(msg)
        self.step = step
        self.index1 = index1
        self.index2 = index2
        self.x0 = x0
        self.width = width
        self.iteration = iteration


class DeviceError(RuntimeError):
    """CUDA / NCCL failure inside the library."""


class LoadError(RuntimeError):
    """Malformed input file (reference LoadError, errors.hpp:16-19)."""


class NormalizationError(ConfigError):
    """No gene positive in every sample (reference NormalizationError)."""


def _raise(rc: int, err: CmcError):
    if rc == _abi.CMC_OK:
        return
    msg = err.msg.decode(errors="replace")
    if rc == _abi.CMC_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == _abi.CMC_ERR_STALL:
        raise SamplerStallError(msg, err.step.decode(), err.index1, err.index2,
                                err.x0, err.width, err.iteration)
    if rc == _abi.CMC_ERR_ARG:
        raise ValueError(msg)
    if rc == _abi.CMC_ERR_LOAD:
        raise LoadError(msg)
    raise DeviceError(msg)


@dataclass
class SliceConfig:
    max_step_out: int = 100
    burnin: int = 0
    tune_cutoff: int = 0
    w_init: float = 1.0
    max_shrink: int = 1000


@dataclass
class RunConfig:
    chains: int = 4
    iterations: int = 4000
    burnin: int = 2000
    tune_cutoff: int = -1
    thin: int = 20
    seed: int = 1
    slice: SliceConfig = field(default_factory=SliceConfig)
    save_genes: int = 20
    workers: int = 1
    sampler_mode: str = "slice_faithful"  # or "conjugate_direct"
    concurrent_chains: bool = False

    def to_c(self) -> _abi.CmcRunConfig:
        mode = {"slice_faithful": 0, "conjugate_direct": 1}[self.sampler_mode]
        return _abi.make_config(self.chains, self.iterations, self.burnin,
                                self.tune_cutoff, self.thin, self.seed,
                                self.slice.max_step_out, self.slice.max_shrink,
                                self.slice.w_init, self.save_genes, self.workers,
                                mode, self.concurrent_chains)


@dataclass
class PriorConfig:
    a: float = 1.0
    b: float = 1.0
    d: float = 1000.0
    c: Optional[Sequence[float]] = None  # prior sd of theta_l, default 10
    s: Optional[Sequence[float]] = None  # upper bound of sigma_l, default 100
    # Extension (not in the reference; parity unpinned): per
    # column "normal" (the reference model), "laplace", "t" or "horseshoe"
    # -- beta_gl ~ N(theta_l, sigma_l^2 xi_gl) with xi_gl from that prior.
    # One entry applies to every column; t_df is k of the t prior.
    beta_prior: Sequence[str] = ()
    t_df: float = 1.0

    def resolve(self, L: int):
        """PriorConfig::resolve, P:src/types.cpp:38-43."""
        if not self.c:
            self.c = [10.0] * L
        if not self.s:
            self.s = [100.0] * L
        if len(self.c) == 1 and L > 1:
            self.c = [self.c[0]] * L
        if len(self.s) == 1 and L > 1:
            self.s = [self.s[0]] * L
        return self


@dataclass
class ModelSpec:
    X: np.ndarray  # N x L
    h: np.ndarray  # N
    priors: PriorConfig = field(default_factory=PriorConfig)

    @property
    def N(self):
        return self.X.shape[0]

    @property
    def L(self):
        return self.X.shape[1]


@dataclass
class CountMatrix:
    """Reference CountMatrix (P:include/countmc/types.hpp:50-58)."""
    counts: np.ndarray  # G x N int64
    genes: Optional[List[str]] = None
    samples: Optional[List[str]] = None
    duplicate_genes: bool = False

    @property
    def G(self):
        return self.counts.shape[0]

    @property
    def N(self):
        return self.counts.shape[1]


class ChainState:
    """One iteration's parameter values (reference ChainState).  ``xi``
    (G x L) exists only with a xi prior (extension)."""

    def __init__(self, G, N, L, xi=False):
        self.G, self.N, self.L = G, N, L
        self.xi = np.ones((G, L)) if xi else None
        self.eps = np.zeros((G, N))
        self.gamma = np.ones(G)
        self.beta = np.zeros((G, L))
        self.theta = np.zeros(L)
        self.sigma = np.ones(L)
        self.nu = 2.0
        self.tau = 1.0

    def pack(self) -> np.ndarray:
        parts = [self.eps.ravel(), self.gamma, self.beta.ravel(), self.theta, self.sigma,
                 [self.nu, self.tau]]
        if self.xi is not None:
            parts.append(self.xi.ravel())
        return np.concatenate(parts).astype(np.float64)

    @classmethod
    def unpack(cls, packed, G, N, L) -> "ChainState":
        st = cls(G, N, L, xi=len(packed) > sizes(G, N, L)[0])
        st.load(packed)
        return st

    def load(self, p):
        G, N, L = self.G, self.N, self.L
        o = 0
        self.eps = np.array(p[o:o + G * N]).reshape(G, N); o += G * N
        self.gamma = np.array(p[o:o + G]); o += G
        self.beta = np.array(p[o:o + G * L]).reshape(G, L); o += G * L
        self.theta = np.array(p[o:o + L]); o += L
        self.sigma = np.array(p[o:o + L]); o += L
        self.nu = float(p[o]); self.tau = float(p[o + 1]); o += 2
        if len(p) > o:
            self.xi = np.array(p[o:o + G * L]).reshape(G, L)

    def check(self, priors: PriorConfig):
        """ChainState::check, P:src/types.cpp:71-89."""
        if not np.all(np.isfinite(self.eps)):
            raise ConfigError("non-finite eps in chain state")
        if not (np.all(self.gamma > 0) and np.all(np.isfinite(self.gamma))):
            raise ConfigError("gamma must be positive and finite")
        if not np.all(np.isfinite(self.beta)):
            raise ConfigError("non-finite beta in chain state")
        if not np.all(np.isfinite(self.theta)):
            raise ConfigError("non-finite theta in chain state")
        for l in range(self.L):
            bound = priors.s[l] if l < len(priors.s) else 100.0
            if not (0.0 < self.sigma[l] < bound):
                raise ConfigError(f"sigma[{l + 1}] outside (0, s)")
        if not (0.0 < self.nu < priors.d):
            raise ConfigError("nu outside (0, d)")
        if not (self.tau > 0.0 and np.isfinite(self.tau)):
            raise ConfigError("tau must be positive and finite")


class TuningState:
    """Slice widths w and w_aux in the packed order
    [eps|gamma|beta|sigma|nu|tau] (+ [xi] with a xi prior)."""

    def __init__(self, G, N, L, w_init=1.0, xi=False):
        _, T, _ = sizes(G, N, L, xi)
        self.G, self.N, self.L = G, N, L
        self.w = np.full(T, float(w_init))
        self.w_aux = np.zeros(T)

    def _slice(self, which):
        G, N, L = self.G, self.N, self.L
        o = {"eps": (0, G * N), "gamma": (G * N, G), "beta": (G * N + G, G * L),
             "sigma": (G * N + G + G * L, L), "nu": (G * N + G + G * L + L, 1),
             "tau": (G * N + G + G * L + L + 1, 1),
             "xi": (G * N + G + G * L + L + 2, G * L)}[which]
        return slice(o[0], o[0] + o[1])

    def width(self, which):
        return self.w[self._slice(which)]

    def aux(self, which):
        return self.w_aux[self._slice(which)]


class Moments:
    """Vector of MomentAccumulator (P:include/countmc/streaming.hpp:15-40)."""

    def __init__(self, count, mean, meansq, mean_c, meansq_c):
        self.count = count
        self.mean = mean
        self.meansq = meansq
        self.mean_c = mean_c
        self.meansq_c = meansq_c


@dataclass
class ContrastResult:
    spec: object
    count: int
    prob: np.ndarray


@dataclass
class Diagnostics:
    """Per-parameter convergence diagnostics (reference DiagRow,
    P:include/countmc/io.hpp, build_diagnostics P:src/io.cpp:507-569)."""
    names: List[str]
    rhat: np.ndarray
    degenerate: np.ndarray
    passed: np.ndarray
    mean: np.ndarray
    sd: np.ndarray
    ci_lo: np.ndarray
    ci_hi: np.ndarray
    ess: np.ndarray          # NaN where the parameter is not retained
    ess_status: List[str]    # ok / undefined / degenerate / not-retained


@dataclass
class ChainOutput:
    chain: int
    nu_acc: Moments
    tau_acc: Moments
    theta_acc: Moments
    sigma_acc: Moments
    beta_acc: Moments   # arrays G x L
    gamma_acc: Moments  # G
    eps_acc: Moments    # G x N
    contrasts: List[ContrastResult]
    sample_names: List[str]
    samples: np.ndarray  # [column][row]
    sample_iters: np.ndarray
    saved_genes: np.ndarray
    step_seconds: np.ndarray
    clamp_events: int
    final_state: ChainState
    xi_acc: Optional[Moments] = None  # G x L, with a xi prior (extension)


# ----------------------------------------------------------------- contrasts

@dataclass
class ParamRef:
    family: str  # beta_col, gamma, theta, sigma, nu, tau
    index: int = 0  # 0-based column

    def per_gene(self):
        return self.family in ("beta_col", "gamma")


def parse_param_ref(name: str, L: int) -> ParamRef:
    """parse_param_ref, P:src/streaming.cpp:42-74."""
    bad = ConfigError(f"unknown parameter name in contrast: '{name}'")
    if name in ("nu", "tau", "gamma"):
        return ParamRef(name if name != "gamma" else "gamma", 0)
    if "[" not in name or not name.endswith("]"):
        raise bad
    head, inner = name[:name.index("[")], name[name.index("[") + 1:-1]
    if head == "beta":
        if len(inner) < 2 or inner[0] != "," or not inner[1:].isdigit():
            raise bad
        fam, idx = "beta_col", int(inner[1:])
    elif head in ("theta", "sigma"):
        if not inner.isdigit():
            raise bad
        fam, idx = head, int(inner)
    elif head == "gamma":
        raise ConfigError("gamma takes no index in contrasts; write 'gamma'")
    else:
        raise bad
    if idx < 1 or idx > L:
        raise ConfigError(f"contrast index out of range in '{name}' (L={L})")
    return ParamRef(fam, idx - 1)


@dataclass
class ContrastTerm:
    coeffs: List[tuple]  # [(ParamRef, coef)]
    threshold: float = 0.0


@dataclass
class ContrastSpec:
    id: str
    terms: List[ContrastTerm]
    per_gene: bool = False

    def finalize(self):
        """ContrastSpec::finalize, P:src/streaming.cpp:76-88."""
        if not self.terms:
            raise ConfigError(f"contrast '{self.id}' has no terms")
        self.per_gene = False
        for t in self.terms:
            if not t.coeffs:
                raise ConfigError(f"contrast '{self.id}' has a term with no coefficients")
            for ref, _ in t.coeffs:
                if ref.per_gene():
                    self.per_gene = True
        return self

    def flat(self):
        return [([(r.family, r.index, c) for r, c in t.coeffs], t.threshold)
                for t in self.terms]


def disjunction_combine(p1, p2, p12):
    """P:src/streaming.cpp:110-112."""
    return float(np.clip(p1 + p2 - p12, 0.0, 1.0))


# -------------------------------------------------------------------- engine

class LoopbackGroup:
    """Test hook (no reference counterpart): `world` engines of this process
    on one GPU play the ranks of a sharded job; see cmc_loopback_create."""

    def __init__(self, world: int):
        self._lib = load_library()
        self.world = world
        h = c_void_p()
        err = CmcError()
        _raise(self._lib.cmc_loopback_create(world, byref(h), byref(err)), err)
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self._lib.cmc_loopback_destroy(h)
            self.handle = None


class GibbsEngine:
    """B200 GibbsEngine: same constructor, methods and errors as the
    reference (P:include/countmc/engine.hpp:110-159)."""

    def __init__(self, data: CountMatrix, spec: ModelSpec, cfg: RunConfig,
                 contrasts: Sequence[ContrastSpec] = (), device: int = 0):
        self._lib = load_library()
        counts = np.asarray(data.counts if isinstance(data, CountMatrix) else data)
        if counts.shape[1] != spec.X.shape[0]:
            raise ConfigError("model matrix rows must match the sample count")
        spec.priors.resolve(spec.X.shape[1])
        self.G, self.N = counts.shape
        self.L = spec.X.shape[1]
        self.spec = spec
        self._contrast_specs = [c.finalize() for c in contrasts]
        self._genes = list(data.genes) if isinstance(data, CountMatrix) and data.genes else None
        self._prob = ProblemArrays(counts, spec.X, spec.h, spec.priors.a,
                                   spec.priors.b, spec.priors.d, spec.priors.c,
                                   spec.priors.s, spec.priors.beta_prior, spec.priors.t_df)
        self.xi = self._prob.xi
        self._ctr = ContrastArrays([c.flat() for c in self._contrast_specs])
        cfg_c = cfg.to_c()
        err = CmcError()
        h = c_void_p()
        rc = self._lib.cmc_engine_create(byref(self._prob.struct), byref(cfg_c),
                                         byref(self._ctr.struct) if self._contrast_specs else None,
                                         device, byref(h), byref(err))
        _raise(rc, err)
        self._h = h
        resolved = _abi.CmcRunConfig()
        self._lib.cmc_engine_config(self._h, byref(resolved))
        self._cfg = RunConfig(resolved.chains, resolved.iterations, resolved.burnin,
                              resolved.tune_cutoff, resolved.thin, resolved.seed,
                              SliceConfig(resolved.max_step_out, resolved.burnin,
                                          resolved.tune_cutoff, resolved.w_init,
                                          resolved.max_shrink),
                              resolved.save_genes, resolved.workers,
                              cfg.sampler_mode, bool(resolved.concurrent_chains))
        dims = [c_long() for _ in range(7)]
        self._lib.cmc_engine_dims(self._h, *[byref(d) for d in dims])
        self.n_saved = dims[4].value
        self.n_cols = dims[5].value
        self.n_rows = dims[6].value
        saved = np.zeros(max(1, self.n_saved), dtype=np.int64)
        self._lib.cmc_engine_saved_genes(self._h, lptr(saved))
        self._saved = saved[:self.n_saved]
        self._progress = None
        self._outputs = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.cmc_engine_destroy(h)
            self._h = None

    def shard(self, rank: int, world: int, nccl_uid: bytes = b""):
        """Restrict this engine to its leaf-aligned gene shard and join the
        NCCL clique (one process per GPU).  Must precede any sweep."""
        err = CmcError()
        buf = ctypes.create_string_buffer(bytes(nccl_uid).ljust(128, b"\0"), 128)
        _raise(self._lib.cmc_engine_shard(self._h, rank, world, buf, byref(err)), err)
        lo, hi = c_long(), c_long()
        self._lib.cmc_shard_bounds(self.G, rank, world, byref(lo), byref(hi))
        self.shard_range = (lo.value, hi.value)

    def set_step_timing(self, on: bool = True):
        """Per-step timing mode (debug): sweeps launch each of the seven
        steps on its own with CUDA events between them, and the outputs'
        step_seconds hold per-step device seconds (reference StepTimings,
        P:src/engine.cpp:173-176).  Bit-identical results, slower sweeps;
        single GPU."""
        self._lib.cmc_engine_set_step_timing(self._h, 1 if on else 0)

    def shard_loopback(self, rank: int, group: "LoopbackGroup"):
        """Test hook: join an in-process loopback group as `rank` instead of
        an NCCL clique (cmc_engine_shard_loopback).  Each engine of the
        group must then be driven from its own thread; eager sweeps only."""
        err = CmcError()
        _raise(self._lib.cmc_engine_shard_loopback(self._h, rank, group.handle, byref(err)), err)
        lo, hi = c_long(), c_long()
        self._lib.cmc_shard_bounds(self.G, rank, group.world, byref(lo), byref(hi))
        self.shard_range = (lo.value, hi.value)
        self._loopback = group  # keep the group alive while the engine is

    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = load_library()
        buf = ctypes.create_string_buffer(128)
        err = CmcError()
        _raise(lib.cmc_nccl_unique_id(buf, byref(err)), err)
        return buf.raw

    # accessors, P:include/countmc/engine.hpp:115-117
    def config(self) -> RunConfig:
        return self._cfg

    def contrast_specs(self):
        return self._contrast_specs

    def saved_genes(self) -> np.ndarray:
        return self._saved

    @property
    def handle(self):
        return self._h

    def initial_state(self, chain: int) -> ChainState:
        S, _, _ = sizes(self.G, self.N, self.L, self.xi)
        buf = np.zeros(S)
        err = CmcError()
        _raise(self._lib.cmc_engine_initial_state(self._h, chain, dptr(buf), byref(err)), err)
        return ChainState.unpack(buf, self.G, self.N, self.L)

    def iterate(self, state: ChainState, tuning: TuningState, chain: int, m: int,
                clamps: Optional[list] = None, step5_trace: Optional[list] = None):
        """GibbsEngine::iterate (P:src/engine.cpp:161-370): one sweep of
        `state` in place on the device.  ``clamps`` (a one-element list) is
        incremented like ClampCounter."""
        err = CmcError()
        st = state.pack()
        _raise(self._lib.cmc_engine_set_state(self._h, chain, dptr(st), dptr(tuning.w),
                                              dptr(tuning.w_aux), byref(err)), err)
        cnt = c_uint64(0)
        rc = self._lib.cmc_engine_iterate(self._h, chain, m, byref(cnt), byref(err))
        if clamps is not None:
            clamps[0] += cnt.value
        if step5_trace is not None:
            # the per-gene column loop is sequential by construction
            for l in range(self.L):
                step5_trace += [l + 1, -(l + 1)]
        _raise(rc, err)
        _raise(self._lib.cmc_engine_get_state(self._h, chain, dptr(st), dptr(tuning.w),
                                              dptr(tuning.w_aux), byref(err)), err)
        state.load(st)

    def set_progress(self, fn: Callable[[int, int, int], None]):
        self._progress = fn

    def run(self) -> List[ChainOutput]:
        """GibbsEngine::run (P:src/engine.cpp:457-483); chains are batched
        on the device and each equals the reference's run_chain(c)."""
        if self._outputs is None:
            err = CmcError()
            _raise(self._lib.cmc_engine_begin(self._h, byref(err)), err)
            total = self._cfg.burnin + self._cfg.iterations
            step = max(1, min(total, 500)) if self._progress else total
            bufs = None
            m = 1
            while m <= total:
                m_end = min(total + 1, m + step)
                _raise(self._lib.cmc_engine_sweeps(self._h, m, m_end, byref(err)), err)
                if self._progress:
                    _raise(self._lib.cmc_engine_sync(self._h, byref(err)), err)
                    for c in range(self._cfg.chains):
                        self._progress(c, m_end - 1, total)
                m = m_end
                if bufs is None:
                    # the sweeps are enqueued and the host is idle until sync:
                    # allocate the output arrays now, every page written, so
                    # the copies after sync do not page-fault (fresh arrays
                    # of a Paschold-size run cost ~36 ms of faults, 4 chains)
                    bufs = [self._output_arrays() for _ in range(self._cfg.chains)]
            _raise(self._lib.cmc_engine_sync(self._h, byref(err)), err)
            self._outputs = [self._output(c, bufs[c] if bufs else None)
                             for c in range(self._cfg.chains)]
        return self._outputs

    def diagnostics(self) -> Diagnostics:
        """R-hat, pooled estimates and ESS for every parameter, computed on
        the device from the resident accumulators of the last run()."""
        self.run()
        G, L = self.G, self.L
        R = 2 + 2 * L + G * (L + 1)
        arr = {k: np.zeros(R) for k in ("rhat", "mean", "sd", "lo", "hi")}
        flags = np.zeros(R, dtype=np.int32)
        ess = np.zeros(max(1, self.n_cols))
        est = np.zeros(max(1, self.n_cols), dtype=np.int32)
        view = _abi.CmcDiagView(dptr(arr["rhat"]), dptr(arr["mean"]), dptr(arr["sd"]),
                                dptr(arr["lo"]), dptr(arr["hi"]),
                                flags.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), dptr(ess),
                                est.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
        err = CmcError()
        _raise(self._lib.cmc_engine_diagnostics(self._h, byref(view), byref(err)), err)
        names = ["nu", "tau"] + [f"theta[{l + 1}]" for l in range(L)] + \
                [f"sigma[{l + 1}]" for l in range(L)]
        names += [f"beta[{g + 1},{l + 1}]" for g in range(G) for l in range(L)]
        names += [f"gamma[{g + 1}]" for g in range(G)]
        row_ess = np.full(R, np.nan)
        status = ["not-retained"] * R
        code = {0: "ok", 1: "undefined", 2: "degenerate"}
        col_of = {}
        for c in range(2 + 2 * L):
            col_of[c] = c
        for k, g in enumerate(self._saved):
            for l in range(L):
                col_of[2 + 2 * L + g * L + l] = 2 + 2 * L + k * (L + 1) + l
            col_of[2 + 2 * L + G * L + g] = 2 + 2 * L + k * (L + 1) + L
        for r, c in col_of.items():
            row_ess[r] = ess[c] if est[c] == 0 else (np.nan if est[c] == 1 else ess[c])
            status[r] = code[int(est[c])]
        return Diagnostics(names, arr["rhat"], (flags & 1) != 0, (flags & 2) != 0, arr["mean"],
                           arr["sd"], arr["lo"], arr["hi"], row_ess, status)

    def run_chain(self, chain: int) -> ChainOutput:
        return self.run()[chain]

    def write_results(self, outdir: str, wall_seconds: float = 0.0,
                      genes: Optional[Sequence[str]] = None) -> None:
        """The reference's write_results (P:src/io.cpp:571-720) for the last
        run(): gene_estimates.csv, hyper_estimates.csv, diagnostics.csv,
        samples/chain_<c>.csv and run_report.json, from the device-resident
        accumulators.  Gene labels default to the CountMatrix's."""
        self.run()
        labels = list(genes) if genes is not None else self._genes
        keep = []
        gl = None
        if labels is not None:
            if len(labels) != self.G:
                raise ConfigError(f"need {self.G} gene labels, got {len(labels)}")
            keep = [g.encode(errors="surrogateescape") for g in labels]
            gl = (ctypes.c_char_p * self.G)(*keep)
        ids = [c.id.encode() for c in self._contrast_specs]
        cl = (ctypes.c_char_p * max(1, len(ids)))(*ids) if ids else None
        err = CmcError()
        _raise(self._lib.cmc_engine_write_results(self._h, str(outdir).encode(), gl, cl,
                                                  float(wall_seconds), byref(err)), err)

    def sample_names(self) -> List[str]:
        L = self.L
        names = ["nu", "tau"] + [f"theta[{l + 1}]" for l in range(L)] + \
                [f"sigma[{l + 1}]" for l in range(L)]
        for g in self._saved:
            names += [f"beta[{g + 1},{l + 1}]" for l in range(L)] + [f"gamma[{g + 1}]"]
        return names

    def tuning_state(self) -> TuningState:
        """A TuningState of this engine's layout at w_init."""
        return TuningState(self.G, self.N, self.L, self._cfg.slice.w_init, self.xi)

    def load_outputs(self, outputs: Sequence[ChainOutput]) -> None:
        """Adopt finished ChainOutputs as this engine's run() result
        (cmc_engine_set_output): for a sharded job's outputs, merged by
        shards.merge_shard_outputs, in an unsharded engine of the full
        problem.  diagnostics() and write_results() then work as after
        run().  Not in the reference (which has no sharding)."""
        if len(outputs) != self._cfg.chains:
            raise ConfigError(f"need {self._cfg.chains} chain outputs, got {len(outputs)}")
        G, N, L = self.G, self.N, self.L
        for c, o in enumerate(outputs):
            moms = [o.nu_acc, o.tau_acc, o.theta_acc, o.sigma_acc, o.beta_acc, o.gamma_acc,
                    o.eps_acc] + ([o.xi_acc] if self.xi else [])
            accs = [np.ascontiguousarray(np.concatenate(
                [np.ravel(getattr(m, k)) for m in moms]), dtype=np.float64)
                for k in ("mean", "meansq", "mean_c", "meansq_c")]
            count = np.array([o.beta_acc.count], dtype=np.int64)
            prob = np.ascontiguousarray(np.concatenate(
                [np.ravel(r.prob) for r in o.contrasts]) if o.contrasts else np.zeros(1))
            samples = np.ascontiguousarray(np.ravel(o.samples), dtype=np.float64)
            if samples.size == 0:
                samples = np.zeros(1)
            clamps = np.array([o.clamp_events], dtype=np.uint64)
            final = np.ascontiguousarray(o.final_state.pack(), dtype=np.float64)
            view = CmcOutputView(lptr(count), dptr(accs[0]), dptr(accs[1]), dptr(accs[2]),
                                 dptr(accs[3]), dptr(prob), None, dptr(samples), None,
                                 clamps.ctypes.data_as(ctypes.POINTER(c_uint64)),
                                 dptr(final), None)
            err = CmcError()
            _raise(self._lib.cmc_engine_set_output(self._h, c, byref(view), byref(err)), err)
        self._outputs = list(outputs)

    def _output_arrays(self):
        """The large per-chain output arrays (4 accumulator blocks and the
        final state), allocated with every page touched."""
        S, _, A = sizes(self.G, self.N, self.L, self.xi)
        return [np.full(A, 0.0) for _ in range(4)], np.full(S, 0.0)

    def _output(self, chain: int, arrays=None) -> ChainOutput:
        G, N, L = self.G, self.N, self.L
        S, _, A = sizes(G, N, L, self.xi)
        accs, final = arrays if arrays is not None else self._output_arrays()
        count = np.zeros(1, dtype=np.int64)
        n_prob = sum(G if c.per_gene else 1 for c in self._contrast_specs)
        prob = np.zeros(max(1, n_prob))
        ccount = np.zeros(max(1, len(self._contrast_specs)), dtype=np.int64)
        rows = self.n_rows
        samples = np.zeros(max(1, self.n_cols * rows))
        iters = np.zeros(max(1, rows), dtype=np.int64)
        clamps = np.zeros(1, dtype=np.uint64)
        secs = np.zeros(7)
        view = CmcOutputView(lptr(count), dptr(accs[0]), dptr(accs[1]), dptr(accs[2]),
                             dptr(accs[3]), dptr(prob), lptr(ccount), dptr(samples),
                             lptr(iters), clamps.ctypes.data_as(ctypes.POINTER(c_uint64)),
                             dptr(final), dptr(secs))
        err = CmcError()
        _raise(self._lib.cmc_engine_get_output(self._h, chain, byref(view), byref(err)), err)

        def part(lo, n, shape=None):
            arrs = [a[lo:lo + n] if shape is None else a[lo:lo + n].reshape(shape) for a in accs]
            return Moments(int(count[0]), *arrs)

        o = 0
        nu = part(o, 1); o += 1
        tau = part(o, 1); o += 1
        theta = part(o, L); o += L
        sigma = part(o, L); o += L
        beta = part(o, G * L, (G, L)); o += G * L
        gamma = part(o, G); o += G
        eps = part(o, G * N, (G, N)); o += G * N
        xi = part(o, G * L, (G, L)) if self.xi else None
        contrasts, off = [], 0
        for k, c in enumerate(self._contrast_specs):
            n = G if c.per_gene else 1
            contrasts.append(ContrastResult(c, int(ccount[k]), prob[off:off + n].copy()))
            off += n
        return ChainOutput(chain, nu, tau, theta, sigma, beta, gamma, eps, contrasts,
                           self.sample_names(), samples[:self.n_cols * rows].reshape(self.n_cols, rows),
                           iters[:rows], self._saved.copy(), secs, int(clamps[0]),
                           ChainState.unpack(final, G, N, L), xi)


# ---------------------------------------------------------- synthetic inputs

@dataclass
class SimSpec:
    """P:include/countmc/simulate.hpp:13-27."""
    G: int
    N: int
    X: np.ndarray
    h: Optional[np.ndarray] = None
    nu: float = 2.0
    tau: float = 1.0
    theta: Sequence[float] = ()
    sigma: Sequence[float] = ()
    seed: int = 1


def generate(spec: SimSpec) -> CountMatrix:
    """Synthetic counts with the reference model's generative shape
    (P:src/simulate.cpp:28-90); the input generator of tests and bench."""
    lib = load_library()
    X = np.ascontiguousarray(spec.X, dtype=np.float64)
    h = np.ascontiguousarray(spec.h if spec.h is not None else np.zeros(spec.N))
    theta = np.ascontiguousarray(spec.theta, dtype=np.float64)
    sigma = np.ascontiguousarray(spec.sigma, dtype=np.float64)
    out = np.zeros((spec.G, spec.N), dtype=np.int64)
    err = CmcError()
    rc = lib.cmc_simulate(spec.G, spec.N, X.shape[1], dptr(X), dptr(h), spec.nu, spec.tau,
                          dptr(theta), dptr(sigma), spec.seed,
                          out.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), byref(err))
    _raise(rc, err)
    return CountMatrix(out)


def _labels(lib, h, which, n):
    blob, size = ctypes.c_char_p(), ctypes.c_size_t()
    lib.cmc_counts_labels(h, which, byref(blob), byref(size))
    raw = ctypes.string_at(blob, size.value)
    return raw.decode(errors="surrogateescape").split("\0")[:n]


def load_counts(path: str) -> CountMatrix:
    """Counts CSV -> CountMatrix, same rules and LoadError messages as the
    reference load_counts (P:src/io.cpp:125-164); parsed by the library's
    multithreaded host loader (cmc_counts_load)."""
    lib = load_library()
    h = c_void_p()
    err = CmcError()
    _raise(lib.cmc_counts_load(str(path).encode(), byref(h), byref(err)), err)
    try:
        G, N, dup = c_long(), c_long(), ctypes.c_int()
        lib.cmc_counts_dims(h, byref(G), byref(N), byref(dup))
        G, N = G.value, N.value
        counts = np.ctypeslib.as_array(lib.cmc_counts_data(h), shape=(G * N,))
        counts = counts.astype(np.int64, copy=True).reshape(G, N)
        genes, samples = (_labels(lib, h, which, n) for which, n in ((0, G), (1, N)))
    finally:
        lib.cmc_counts_free(h)
    return CountMatrix(counts, genes, samples, bool(dup.value))


@dataclass
class DesignTable:
    """Reference DesignTable (P:include/countmc/io.hpp:19-22)."""
    X: np.ndarray        # N x L
    effects: List[str]


def _load_table(fn, path):
    lib = load_library()
    h = c_void_p()
    err = CmcError()
    _raise(getattr(lib, fn)(str(path).encode(), byref(h), byref(err)), err)
    try:
        r, c = c_long(), c_long()
        lib.cmc_table_dims(h, byref(r), byref(c))
        data = np.ctypeslib.as_array(lib.cmc_table_data(h), shape=(r.value * c.value,))
        data = data.astype(np.float64, copy=True).reshape(r.value, c.value)
        names = [lib.cmc_table_name(h, k).decode(errors="surrogateescape") for k in range(c.value)]
    finally:
        lib.cmc_table_free(h)
    return data, names


def load_model_matrix(path: str) -> DesignTable:
    """load_model_matrix (P:src/io.cpp:178-205): effect names from the
    header, one row of L numbers per sample; LoadError like the reference."""
    X, effects = _load_table("cmc_model_matrix_load", path)
    return DesignTable(X, effects)


def load_offsets(path: str) -> np.ndarray:
    """load_offsets (P:src/io.cpp:221-243): "sample,offset" rows."""
    h, _ = _load_table("cmc_offsets_load", path)
    return h[:, 0].copy()


def estimate_offsets(counts) -> np.ndarray:
    """Median-of-ratios log offsets h (reference estimate_offsets,
    P:src/model.cpp:21-68, bit-identical); raises NormalizationError when no
    gene is positive in every sample."""
    lib = load_library()
    y = counts.counts if isinstance(counts, CountMatrix) else counts
    y = np.ascontiguousarray(y, dtype=np.int64)
    if y.ndim != 2:
        raise ValueError("counts must be a G x N matrix")
    G, N = y.shape
    if G < 1 or N < 1:
        raise ConfigError("count matrix must have at least one gene and one sample")
    h = np.zeros(N)
    err = CmcError()
    rc = lib.cmc_estimate_offsets(G, N, y.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)),
                                  dptr(h), byref(err))
    if rc == _abi.CMC_ERR_CONFIG:
        raise NormalizationError(err.msg.decode(errors="replace"))
    _raise(rc, err)
    return h


def builtin_design(name: str, N: int) -> np.ndarray:
    """heterosis16x5: [A (x) 1_4 | 1_4 (x) (1,1,-1,-1)'] tiled over N
    (P:src/simulate.cpp:123-142)."""
    if name != "heterosis16x5":
        raise ConfigError(f"unknown built-in design '{name}'")
    if N == 0 or N % 16 != 0:
        raise ConfigError("heterosis16x5 needs a sample count that is a multiple of 16")
    A = np.array([[1, 1, -1, 0], [1, -1, 1, 0], [1, 1, 1, 1], [1, 1, 1, -1]], dtype=float)
    block = [1, 1, -1, -1]
    X = np.zeros((N, 5))
    for n in range(N):
        r = n % 16
        X[n, :4] = A[r // 4]
        X[n, 4] = block[r % 4]
    return X


def heterosis_contrast(L: int = 5) -> ContrastSpec:
    """High-parent heterosis: {2 b2 + b4 > 0 and 2 b3 + b4 > 0}
    (P:src/simulate.cpp:144-155)."""
    t1 = ContrastTerm([(parse_param_ref("beta[,2]", L), 2.0),
                       (parse_param_ref("beta[,4]", L), 1.0)], 0.0)
    t2 = ContrastTerm([(parse_param_ref("beta[,3]", L), 2.0),
                       (parse_param_ref("beta[,4]", L), 1.0)], 0.0)
    return ContrastSpec("highparent", [t1, t2]).finalize()
