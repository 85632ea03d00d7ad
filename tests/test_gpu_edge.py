"""GPU: edge shapes the heterosis bench never reaches, each bit-for-bit
against the oracle (θ to 1e-12), the way the reference's own tests probe
them (P:tests/test_engine.cpp, test_model.cpp clamp semantics):

* continuous covariates: up to N distinct values per model-matrix column,
  so the generic gene kernel (group sums in shared memory) runs;
* L = 16, the widest model matrix this build supports;
* the exp(700) clamp: offsets push h + xb + ε past 700, and the clamp
  counts must agree too;
* ragged G (not a multiple of the 128-gene block or the 1024-gene leaf)."""
import numpy as np
import pytest

import oracle
from paper_1606_06659_b200 import _abi

from helpers import Product, advance, mismatch, packed_start

pytestmark = pytest.mark.gpu


def _sim(G, X, h, seed):
    from paper_1606_06659_b200 import SimSpec, generate
    L = X.shape[1]
    rng = np.random.default_rng(seed)
    theta = np.concatenate([[2.0], rng.normal(0, 0.2, L - 1)])
    sigma = np.full(L, 0.3)
    return generate(SimSpec(G=G, N=X.shape[0], X=X, h=h, nu=8.0, tau=0.7, theta=list(theta),
                            sigma=list(sigma), seed=seed)).counts


def _pair_sweeps(counts, X, h, cfg, sweeps, start=1, chain=0):
    orc = oracle.OracleEngine(counts, X, h, cfg)
    gpu = Product(counts, X, h, cfg)
    st, tw, ta = packed_start(orc, chain, cfg.w_init)
    if start > 1:
        advance(orc, st, tw, ta, chain, 1, start)
    g = [st.copy(), tw.copy(), ta.copy()]
    G, N = counts.shape
    L = X.shape[1]
    th0 = G * N + G + G * L
    clamps = 0
    for m in range(start, start + sweeps):
        c1 = orc.iterate(st, tw, ta, chain, m)
        c2 = gpu.iterate(*g, chain, m)
        assert c1 == c2, f"clamps m={m}: {c1} vs {c2}"
        clamps += c1
        bad = [i for i in mismatch(g[0], st) if not th0 <= i < th0 + L]
        assert not bad, f"m={m}: {bad[:8]}"
        np.testing.assert_allclose(g[0][th0:th0 + L], st[th0:th0 + L], rtol=1e-12, atol=0)
        assert not len(mismatch(g[1], tw)) and not len(mismatch(g[2], ta))
    return clamps


def test_continuous_covariates_generic_group_path():
    rng = np.random.default_rng(3)
    N = 12
    X = np.column_stack([np.ones(N), rng.normal(size=N), rng.uniform(-1, 1, size=N)])
    h = rng.normal(0, 0.1, size=N)
    counts = _sim(700, X, h, 3)
    cfg = _abi.make_config(chains=1, burnin=30, iterations=30, thin=10, seed=4, save_genes=5)
    _pair_sweeps(counts, X, h, cfg, 6)
    _pair_sweeps(counts, X, h, cfg, 3, start=25)


def test_widest_model_matrix():
    rng = np.random.default_rng(5)
    N, L = 24, 16
    X = np.column_stack([np.ones(N), rng.choice([-1.0, 0.0, 1.0], size=(N, L - 1))])
    assert np.linalg.matrix_rank(X) == L
    counts = _sim(300, X, np.zeros(N), 5)
    cfg = _abi.make_config(chains=1, burnin=20, iterations=20, thin=10, seed=6, save_genes=3)
    _pair_sweeps(counts, X, np.zeros(N), cfg, 5)


@pytest.mark.parametrize("w_init", [1000.0, 690.0])
def test_exp_clamp_path_counts_agree(w_init):
    """A first slice interval of width 1000 (w_init) puts step-out bounds and
    shrink proposals past h + xb + eps = 700, where clamped_exp returns
    exp(700) and bumps the ClampCounter (P:src/model.cpp:13-19); the device's
    counts equal the oracle's sweep by sweep.  (Offsets near 700 instead make
    every density ~1e303, which absorbs log(u) and stalls the reference too.)
    Width 690 is within the carried step-out's range but puts the left end
    of some intervals (placement draw u > ~0.97) below exp's normal range, so the ε step-out takes its
    fresh-exp path on one side and a carried exp on the other."""
    from paper_1606_06659_b200 import builtin_design
    X = builtin_design("heterosis16x5", 16)
    counts = _sim(500, X, np.zeros(16), 7)
    cfg = _abi.make_config(chains=1, burnin=20, iterations=20, thin=10, seed=8, save_genes=3,
                           w_init=w_init)
    clamps = _pair_sweeps(counts, X, np.zeros(16), cfg, 4)
    if w_init > 700.0:
        assert clamps > 0


@pytest.mark.parametrize("G", [1, 127, 129, 1023, 1025, 2049])
def test_ragged_gene_counts_run(G):
    """run() with batched chains at block/leaf boundaries: every chain equals
    the oracle's run_chain."""
    from paper_1606_06659_b200 import builtin_design
    X = builtin_design("heterosis16x5", 16)
    counts = _sim(G, X, np.zeros(16), 11)
    cfg = _abi.make_config(chains=2, burnin=20, iterations=20, thin=5, seed=9,
                           save_genes=min(4, G))
    outs = Product(counts, X, np.zeros(16), cfg).run()
    N, L = 16, 5
    th0 = G * N + G + G * L
    for c in range(2):
        o = oracle.OracleEngine(counts, X, np.zeros(16), cfg).run_chain(c)
        bad = [i for i in mismatch(outs[c]["final"], o["final"]) if not th0 <= i < th0 + L]
        assert not bad, (G, c, bad[:5])
        for k in ("mean", "meansq"):
            badk = [i for i in mismatch(outs[c][k], o[k]) if not 2 <= i < 2 + L]
            assert not badk, (G, c, k, badk[:5])


def _run_vs_oracle(counts, X, h, cfg, contrasts=(), priors=None, chains=None):
    outs = Product(counts, X, h, cfg, contrasts=list(contrasts), priors=priors).run()
    G, N = counts.shape
    L = X.shape[1]
    th0 = G * N + G + G * L
    orc = oracle.OracleEngine(counts, X, h, cfg, contrasts=list(contrasts), priors=priors)
    for c in range(chains or cfg.chains):
        o = orc.run_chain(c)
        bad = [i for i in mismatch(outs[c]["final"], o["final"]) if not th0 <= i < th0 + L]
        assert not bad, (c, bad[:5])
        for k in ("mean", "meansq"):
            badk = [i for i in mismatch(outs[c][k], o[k]) if not 2 <= i < 2 + L]
            assert not badk, (c, k, badk[:5])
        assert not len(mismatch(outs[c]["prob"], o["prob"])), c
    return outs


def test_xi_priors_widest_matrix_and_generic_groups():
    rng = np.random.default_rng(21)
    N, L = 24, 16
    X = np.column_stack([np.ones(N), rng.normal(size=(N, L - 1))])   # continuous: J = N
    counts = _sim(200, X, np.zeros(N), 21)
    pri = {"beta_prior": ["normal", "laplace", "t", "horseshoe"] * 4, "t_df": 4.0}
    cfg = _abi.make_config(chains=2, burnin=10, iterations=10, thin=5, seed=2, save_genes=2)
    _run_vs_oracle(counts, X, np.zeros(N), cfg, priors=pri)


def test_eight_contrasts_every_scope():
    from paper_1606_06659_b200 import builtin_design
    X = builtin_design("heterosis16x5", 16)
    counts = _sim(300, X, np.zeros(16), 23)
    cons = [
        [([("beta_col", 1, 2.0), ("beta_col", 3, 1.0)], 0.0),
         ([("beta_col", 2, 2.0), ("beta_col", 3, 1.0)], 0.0)],
        [([("beta_col", 1, 1.0)], 0.1)],
        [([("gamma", 0, 1.0)], 0.5)],
        [([("theta", 1, 1.0), ("sigma", 0, -1.0)], 0.0)],
        [([("nu", 0, 1.0)], 5.0)],
        [([("tau", 0, 1.0)], 0.5), ([("sigma", 2, 1.0)], 0.1)],
        [([("beta_col", 4, 1.0), ("gamma", 0, -0.1)], -0.2)],
        [([("beta_col", 0, 1.0), ("theta", 0, -1.0)], 0.0)],
    ]
    cfg = _abi.make_config(chains=2, burnin=20, iterations=30, thin=10, seed=4, save_genes=3)
    _run_vs_oracle(counts, X, np.zeros(16), cfg, contrasts=cons)


@pytest.mark.parametrize("kw", [
    dict(G=1, chains=4, save_genes=20),              # one gene, both lanes, save > G
    dict(G=60, chains=2, thin=50, iterations=20),    # thin > iterations: no sample rows
    dict(G=60, chains=2, burnin=1),                  # tune_cutoff resolves to 0
    dict(G=200, chains=8),                           # lanes of 4 chains
])
def test_run_configuration_corners(kw):
    from paper_1606_06659_b200 import builtin_design
    G = kw.pop("G")
    X = builtin_design("heterosis16x5", 16)
    counts = _sim(G, X, np.zeros(16), 29)
    args = dict(chains=2, burnin=20, iterations=20, thin=5, seed=6, save_genes=4)
    args.update(kw)
    cfg = _abi.make_config(**args)
    _run_vs_oracle(counts, X, np.zeros(16), cfg,
                   contrasts=[[([("beta_col", 1, 1.0)], 0.0)]])


def test_conjugate_direct_with_xi_prior():
    """gamma/tau by direct draws (1e-12, Marsaglia-Tsang through pow/log) with
    a Laplace xi column; everything slice-sampled stays bit-identical."""
    from paper_1606_06659_b200 import builtin_design
    X = builtin_design("heterosis16x5", 16)
    counts = _sim(300, X, np.zeros(16), 31)
    cfg = _abi.make_config(chains=1, burnin=20, iterations=20, thin=10, seed=3,
                           sampler_mode=_abi.CMC_CONJUGATE_DIRECT)
    pri = {"beta_prior": ["normal", "laplace", "normal", "normal", "normal"]}
    orc = oracle.OracleEngine(counts, X, np.zeros(16), cfg, priors=pri)
    gpu = Product(counts, X, np.zeros(16), cfg, priors=pri)
    st, tw, ta = packed_start(orc, 0)
    g = [st.copy(), tw.copy(), ta.copy()]
    for m in range(1, 5):
        orc.iterate(st, tw, ta, 0, m)
        gpu.iterate(*g, 0, m)
    np.testing.assert_allclose(g[0], st, rtol=1e-9, atol=1e-12)


@pytest.mark.usefixtures("ref")
def test_diagnostics_at_the_chain_limit():
    """32 chains (the device diagnostics' limit) against the reference's
    build_diagnostics numerics."""
    from paper_1606_06659_b200 import CountMatrix, GibbsEngine, ModelSpec, RunConfig, builtin_design
    X = builtin_design("heterosis16x5", 16)
    counts = _sim(40, X, np.zeros(16), 33)
    cfg = RunConfig(chains=32, burnin=20, iterations=20, thin=5, seed=5, save_genes=2)
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(16)), cfg)
    d = eng.diagnostics()
    ref = oracle.RefEngine(counts, X, np.zeros(16), cfg.to_c()).diagnostics(eng.n_cols)
    L = 5
    keep = np.ones(len(d.rhat), bool)
    keep[2:2 + L] = False
    assert not len(mismatch(d.rhat[keep], ref["rhat"][keep]))
    assert not len(mismatch(d.mean[keep], ref["mean"][keep]))


def test_sample_count_at_the_shared_memory_limit():
    """N = 222, the build maximum: the gene kernel's lp block takes
    222 x 128 x 8 B = 222 KB of shared memory beside its static 4.3 KB (one
    block per SM, opt-in); still bit-identical."""
    from helpers import two_col_design
    X = two_col_design(222)
    counts = _sim(150, X, np.zeros(222), 41)
    cfg = _abi.make_config(chains=1, burnin=10, iterations=10, thin=5, seed=2, save_genes=2)
    _pair_sweeps(counts, X, np.zeros(222), cfg, 2)
