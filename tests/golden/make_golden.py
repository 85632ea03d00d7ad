"""Regenerate tests/golden/*.npz from the UNMODIFIED reference library
(oracle/_ref/libcountmc_ref.so, compiled from /root/reference by
oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py

Each fixture holds its own inputs (counts, X, h, config), so the tests do not
depend on any data generator.  Outputs are the reference's own: sweeps from
GibbsEngine::iterate (P:src/engine.cpp:161-370) and run() outputs
(P:src/engine.cpp:378-483).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from paper_1606_06659_b200 import _abi  # noqa: E402
from paper_1606_06659_b200._abi import sizes  # noqa: E402

HETEROSIS = [([("beta_col", 1, 2.0), ("beta_col", 3, 1.0)], 0.0),
             ([("beta_col", 2, 2.0), ("beta_col", 3, 1.0)], 0.0)]


def counts_poisson(G, N, X, theta, seed):
    """Plain numpy inputs (the generator is irrelevant: counts are stored)."""
    rng = np.random.default_rng(seed)
    beta = theta + 0.3 * rng.standard_normal((G, X.shape[1]))
    eps = 0.4 * rng.standard_normal((G, N))
    lam = np.exp(beta @ X.T + eps)
    return rng.poisson(lam).astype(np.int64)


def sweeps_fixture(name, counts, X, h, cfg_kw, chain, m0, m1):
    cfg = _abi.make_config(**cfg_kw)
    ref = oracle.RefEngine(counts, X, h, cfg)
    G, N = counts.shape
    L = X.shape[1]
    _, T, _ = sizes(G, N, L)
    st = ref.initial_state(chain)
    tw, ta = np.full(T, cfg.w_init), np.zeros(T)
    init = st.copy()
    states, tws, tas, clamps = [], [], [], []
    for m in range(m0, m1):
        clamps.append(ref.iterate(st, tw, ta, chain, m))
        states.append(st.copy())
        tws.append(tw.copy())
        tas.append(ta.copy())
    np.savez_compressed(os.path.join(HERE, name), counts=counts, X=X, h=h,
                        cfg=np.array([cfg_kw[k] for k in CFG_KEYS], dtype=np.float64),
                        chain=chain, m0=m0, m1=m1, init=init, states=np.array(states),
                        tw=np.array(tws), ta=np.array(tas), clamps=np.array(clamps, np.uint64),
                        saved=ref.saved_genes())


def run_fixture(name, counts, X, h, cfg_kw, contrasts):
    cfg = _abi.make_config(**cfg_kw)
    ref = oracle.RefEngine(counts, X, h, cfg, contrasts=contrasts)
    outs = ref.run()
    arrays = {}
    for c, o in enumerate(outs):
        for k in ("count", "mean", "meansq", "prob", "samples", "iters", "clamps", "final"):
            arrays[f"c{c}_{k}"] = o[k]
    np.savez_compressed(os.path.join(HERE, name), counts=counts, X=X, h=h,
                        cfg=np.array([cfg_kw[k] for k in CFG_KEYS], dtype=np.float64),
                        saved=ref.saved_genes(), **arrays)


CFG_KEYS = ["chains", "iterations", "burnin", "tune_cutoff", "thin", "seed",
            "max_step_out", "max_shrink", "w_init", "save_genes", "sampler_mode"]


def cfg(**kw):
    base = dict(chains=1, iterations=50, burnin=30, tune_cutoff=-1, thin=10, seed=7,
                max_step_out=100, max_shrink=1000, w_init=1.0, save_genes=8, sampler_mode=0)
    base.update(kw)
    return base


def main():
    X16 = oracle.heterosis16x5(16)
    h16 = np.zeros(16)
    c = counts_poisson(40, 16, X16, np.array([2.5, .2, .2, 0, .1]), 11)
    sweeps_fixture("sweeps_heterosis_g40.npz", c, X16, h16, cfg(chains=3, burnin=20, seed=3),
                   chain=2, m0=1, m1=6)
    sweeps_fixture("sweeps_tiny.npz", np.zeros((1, 1), np.int64), np.ones((1, 1)), np.zeros(1),
                   cfg(burnin=100, iterations=900, tune_cutoff=10, seed=17), chain=0, m0=1, m1=41)
    X4 = np.array([[1, 1], [1, 1], [1, -1], [1, -1]], float)
    c4 = counts_poisson(16, 4, X4, np.array([2.0, 0.5]), 5)
    sweeps_fixture("sweeps_twocol_direct.npz", c4, X4, np.array([0.1, -0.1, 0.05, -0.05]),
                   cfg(burnin=10, tune_cutoff=2, sampler_mode=1), chain=1, m0=1, m1=8)
    c24 = counts_poisson(24, 16, X16, np.array([2.5, .2, .2, 0, .1]), 8)
    run_fixture("run_heterosis_g24.npz", c24, X16, h16,
                cfg(chains=2, burnin=20, iterations=30, thin=5, seed=17, save_genes=6),
                [HETEROSIS])
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
