"""The C restatement against the compiled, unmodified reference (oracle/_ref),
bit for bit, on fresh inputs: sweeps from arbitrary states, both sampler
modes, every contrast scope, stalls and configuration errors.  CPU only;
skipped when oracle/_ref is absent."""
import numpy as np
import pytest

import oracle
from paper_1606_06659_b200 import _abi
from paper_1606_06659_b200._abi import sizes

pytestmark = pytest.mark.usefixtures("ref")


def poisson_counts(G, N, X, seed, scale=0.3):
    rng = np.random.default_rng(seed)
    beta = np.r_[2.0, np.zeros(X.shape[1] - 1)] + scale * rng.standard_normal((G, X.shape[1]))
    return rng.poisson(np.exp(beta @ X.T + 0.4 * rng.standard_normal((G, N)))).astype(np.int64)


def pair(counts, X, h, cfg, contrasts=(), priors=None):
    return (oracle.OracleEngine(counts, X, h, cfg, contrasts=contrasts, priors=priors),
            oracle.RefEngine(counts, X, h, cfg, contrasts=contrasts, priors=priors))


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("G,N,design", [(50, 16, "het"), (7, 4, "two"), (300, 32, "het")])
def test_sweeps_bitwise(G, N, design, mode):
    X = oracle.heterosis16x5(N) if design == "het" else np.array(
        [[1, 1], [1, 1], [1, -1], [1, -1]], float)
    counts = poisson_counts(G, N, X, G + N)
    h = np.linspace(-0.2, 0.2, N)
    cfg = _abi.make_config(chains=2, burnin=15, iterations=20, seed=11, sampler_mode=mode,
                           tune_cutoff=3)
    o, r = pair(counts, X, h, cfg)
    _, T, _ = sizes(G, N, X.shape[1])
    for chain in (0, 1):
        s1 = o.initial_state(chain)
        s2 = r.initial_state(chain)
        assert np.array_equal(s1, s2)
        t1, a1 = np.ones(T), np.zeros(T)
        t2, a2 = t1.copy(), a1.copy()
        for m in range(1, 21):
            c1 = o.iterate(s1, t1, a1, chain, m)
            c2 = r.iterate(s2, t2, a2, chain, m)
            assert np.array_equal(s1, s2), (chain, m)
            assert np.array_equal(t1, t2) and np.array_equal(a1, a2) and c1 == c2


def test_worker_count_does_not_change_reference_bits():
    """P:tests/test_engine.cpp:101-114 on the reference itself, which is what
    makes a sequential restatement a valid oracle."""
    X = oracle.heterosis16x5(16)
    counts = poisson_counts(200, 16, X, 3)
    cfg = _abi.make_config(chains=1, burnin=10, iterations=10, seed=5)
    base = oracle.RefEngine(counts, X, np.zeros(16), cfg, workers=1)
    many = oracle.RefEngine(counts, X, np.zeros(16), cfg, workers=8)
    _, T, _ = sizes(200, 16, 5)
    s1, s2 = base.initial_state(0), many.initial_state(0)
    t1, a1, t2, a2 = np.ones(T), np.zeros(T), np.ones(T), np.zeros(T)
    for m in range(1, 8):
        base.iterate(s1, t1, a1, 0, m)
        many.iterate(s2, t2, a2, 0, m)
    assert np.array_equal(s1, s2)


def test_run_with_every_contrast_scope():
    X = oracle.heterosis16x5(16)
    counts = poisson_counts(30, 16, X, 9)
    contrasts = [
        [([("beta_col", 1, 2.0), ("beta_col", 3, 1.0)], 0.0),
         ([("beta_col", 2, 2.0), ("beta_col", 3, 1.0)], 0.0)],       # heterosis, per gene
        [([("nu", 0, 1.0), ("tau", 0, -1.0)], 0.0)],                 # global
        [([("gamma", 0, 1.0)], 0.5)],                                # per gene gamma
        [([("beta_col", 1, 1.0), ("theta", 1, -1.0)], 0.0)],         # per gene with hyper ref
    ]
    cfg = _abi.make_config(chains=2, burnin=20, iterations=40, thin=4, seed=2, save_genes=5)
    o, r = pair(counts, X, np.zeros(16), cfg, contrasts=contrasts)
    ro = [o.run_chain(c) for c in range(2)]
    rr = r.run()
    for c in range(2):
        for k in ("count", "mean", "meansq", "prob", "ccount", "samples", "iters", "clamps",
                  "final"):
            assert np.array_equal(ro[c][k], rr[c][k]), (c, k)


def test_stall_matches_reference():
    X = np.array([[1, 1], [1, 1], [1, -1], [1, -1]], float)
    counts = poisson_counts(8, 4, X, 11)
    cfg = _abi.make_config(chains=1, burnin=50, iterations=50, seed=17, max_shrink=1,
                           tune_cutoff=5)
    o, r = pair(counts, X, np.zeros(4), cfg)
    with pytest.raises(oracle.StallError) as eo:
        o.run_chain(0)
    with pytest.raises(oracle.StallError) as er:
        r.run()
    a, b = eo.value, er.value
    assert (a.step, a.index1, a.index2, a.iteration, a.x0, a.width) == \
        (b.step, b.index1, b.index2, b.iteration, b.x0, b.width)
    assert str(a) == str(b)


@pytest.mark.parametrize("kw", [dict(tune_cutoff=100, burnin=100), dict(thin=0),
                                dict(workers=0), dict(chains=0), dict(max_shrink=0),
                                dict(w_init=0.0), dict(iterations=0)])
def test_config_validation_matches_reference(kw):
    """P:tests/test_engine.cpp:263-286"""
    X = np.ones((1, 1))
    base = dict(chains=1, burnin=100, iterations=100, seed=17)
    base.update(kw)
    cfg = _abi.make_config(**base)
    with pytest.raises(oracle.ConfigErr):
        oracle.OracleEngine(np.zeros((1, 1), np.int64), X, np.zeros(1), cfg)
    with pytest.raises(oracle.ConfigErr):
        oracle.RefEngine(np.zeros((1, 1), np.int64), X, np.zeros(1), cfg)
