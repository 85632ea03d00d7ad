"""Shared fixtures: problems shaped like the reference's test fixtures
(P:tests/test_engine.cpp:21-64, acceptance c7 P:tests/acceptance/acceptance.cpp:407-430)
and a packed-array driver of the product C-ABI that mirrors oracle.OracleEngine."""
from __future__ import annotations

from ctypes import byref, c_uint64, c_void_p

import numpy as np

from paper_1606_06659_b200 import _abi, builtin_design, generate, SimSpec
from paper_1606_06659_b200._abi import CmcError, ContrastArrays, ProblemArrays, dptr, sizes


def tiny():
    """G = N = L = 1, zero count (P:tests/test_engine.cpp:21-30)."""
    return np.zeros((1, 1), np.int64), np.ones((1, 1)), np.zeros(1)


def two_col_design(N):
    X = np.zeros((N, 2))
    X[:, 0] = 1.0
    X[:, 1] = [1.0 if n < N // 2 else -1.0 for n in range(N)]
    return X


def simulated(G, N, seed):
    """2-column design of P:tests/test_engine.cpp:32-52."""
    X = two_col_design(N)
    data = generate(SimSpec(G=G, N=N, X=X, nu=3.0, tau=0.5, theta=[2.0, 0.5],
                            sigma=[0.5, 0.3], seed=seed))
    return data.counts, X, np.zeros(N)


def heterosis(G, N=16, seed=99):
    """heterosis16x5 data with the c7 hyperparameters."""
    X = builtin_design("heterosis16x5", N)
    data = generate(SimSpec(G=G, N=N, X=X, nu=8.0, tau=0.7,
                            theta=[2.5, 0.2, 0.2, 0.0, 0.1],
                            sigma=[0.4, 0.25, 0.25, 0.15, 0.2], seed=seed))
    return data.counts, X, np.zeros(N)


HETEROSIS = [([("beta_col", 1, 2.0), ("beta_col", 3, 1.0)], 0.0),
             ([("beta_col", 2, 2.0), ("beta_col", 3, 1.0)], 0.0)]


class Product:
    """The CUDA engine through the C-ABI with the oracle's packed API."""

    def __init__(self, counts, X, h, cfg, contrasts=(), priors=None, device=0):
        self.lib = _abi.load_library()
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
        err = CmcError()
        h_ = c_void_p()
        rc = self.lib.cmc_engine_create(byref(self.prob.struct), byref(cfg),
                                        byref(self.ctr.struct) if self.contrasts else None,
                                        device, byref(h_), byref(err))
        if rc:
            raise RuntimeError(err.msg.decode())
        self.h = h_

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.cmc_engine_destroy(self.h)

    def shard_loopback(self, rank, group):
        """Join an in-process loopback group (cmc_engine_shard_loopback)."""
        from ctypes import c_long
        err = CmcError()
        rc = self.lib.cmc_engine_shard_loopback(self.h, rank, group.handle, byref(err))
        if rc:
            raise RuntimeError(err.msg.decode())
        lo, hi = c_long(), c_long()
        self.lib.cmc_shard_bounds(self.G, rank, group.world, byref(lo), byref(hi))
        self.shard_range = (lo.value, hi.value)
        self.group = group

    def initial_state(self, chain):
        S, _, _ = sizes(self.G, self.N, self.L, self.xi)
        st = np.zeros(S)
        err = CmcError()
        assert self.lib.cmc_engine_initial_state(self.h, chain, dptr(st), byref(err)) == 0
        return st

    def saved_genes(self):
        from ctypes import c_long
        dims = [c_long() for _ in range(7)]
        self.lib.cmc_engine_dims(self.h, *[byref(d) for d in dims])
        out = np.zeros(max(1, dims[4].value), np.int64)
        self.lib.cmc_engine_saved_genes(self.h, out.ctypes.data_as(__import__("ctypes").POINTER(c_long)))
        return out[:dims[4].value]

    def iterate(self, st, tw, ta, chain, m):
        err = CmcError()
        rc = self.lib.cmc_engine_set_state(self.h, chain, dptr(st), dptr(tw), dptr(ta), byref(err))
        assert rc == 0, err.msg
        cl = c_uint64(0)
        rc = self.lib.cmc_engine_iterate(self.h, chain, m, byref(cl), byref(err))
        rc2 = self.lib.cmc_engine_get_state(self.h, chain, dptr(st), dptr(tw), dptr(ta), byref(err))
        assert rc2 == 0, err.msg
        if rc:
            import oracle
            raise oracle.StallError(err) if rc == _abi.CMC_ERR_STALL else RuntimeError(err.msg.decode())
        return cl.value

    def run(self):
        import oracle
        err = CmcError()
        rc = self.lib.cmc_engine_run(self.h, byref(err))
        if rc:
            raise oracle.StallError(err) if rc == _abi.CMC_ERR_STALL else RuntimeError(err.msg.decode())
        n_prob = sum(self.G if any(f in ("beta_col", "gamma") for t in c for f, _, _ in t[0])
                     else 1 for c in self.contrasts)
        from ctypes import c_long
        dims = [c_long() for _ in range(7)]
        self.lib.cmc_engine_dims(self.h, *[byref(d) for d in dims])
        n_saved, n_rows = dims[4].value, dims[6].value
        outs = []
        for c in range(self.cfg.chains):
            o, view = oracle.new_outputs(self.G, self.N, self.L, n_saved, n_rows, n_prob,
                                         len(self.contrasts), self.xi)
            rc = self.lib.cmc_engine_get_output(self.h, c, byref(view), byref(err))
            assert rc == 0, err.msg
            outs.append(o)
        return outs


def packed_start(engine_like, chain, w_init=1.0):
    st = engine_like.initial_state(chain)
    G, N, L = engine_like.G, engine_like.N, engine_like.L
    _, T, _ = sizes(G, N, L, getattr(engine_like, "xi", False))
    return st, np.full(T, w_init), np.zeros(T)


def advance(eng, st, tw, ta, chain, m0, m1):
    """Run sweeps m0..m1-1 on packed arrays; returns clamp total."""
    c = 0
    for m in range(m0, m1):
        c += eng.iterate(st, tw, ta, chain, m)
    return c


def mismatch(a, b):
    """Indices where two float arrays differ bitwise (NaN-safe)."""
    a = np.asarray(a)
    b = np.asarray(b)
    return np.flatnonzero(a.view(np.uint64) != b.view(np.uint64)) if a.dtype == np.float64 \
        else np.flatnonzero(a != b)
