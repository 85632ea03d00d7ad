"""The C-ABI library without a GPU: it loads, exports every symbol the
header declares, and its host-side logic (validation, configuration
resolution, saved-gene selection, initial states, shard bounds, synthetic
data) matches the oracle.  No sweep runs here (that needs the device)."""
import os
import re
from ctypes import byref, c_long

import numpy as np
import pytest

import oracle
from paper_1606_06659_b200 import (ConfigError, CountMatrix, GibbsEngine, ModelSpec,
                                   RunConfig, SimSpec, _abi, builtin_design, generate,
                                   heterosis_contrast, parse_param_ref)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "countmc_b200.h")).read()
    return sorted(set(re.findall(r"\b(cmc_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _abi.load_library()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_abi.EXPORTS)
    assert b"sm_100a" in lib.cmc_version()


def test_library_is_in_tree_and_fails_loudly_when_missing(tmp_path):
    assert _abi.LIB_PATH.startswith(ROOT)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _abi._LIB, saved = None, _abi._LIB
        try:
            _abi.load_library(str(tmp_path / "missing.so"))
        finally:
            _abi._LIB = saved


def small(G=64, N=16, seed=4):
    X = builtin_design("heterosis16x5", N)
    c = generate(SimSpec(G=G, N=N, X=X, nu=8, tau=0.7, theta=[2.5, .2, .2, 0, .1],
                         sigma=[.4, .25, .25, .15, .2], seed=seed)).counts
    return c, X, np.zeros(N)


def test_initial_states_and_saved_genes_match_oracle():
    counts, X, h = small()
    for seed in (1, 3, 99):
        cfg = RunConfig(chains=3, burnin=20, iterations=20, seed=seed, save_genes=10)
        eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg)
        orc = oracle.OracleEngine(counts, X, h, cfg.to_c())
        assert np.array_equal(eng.saved_genes(), orc.saved_genes())
        for chain in range(3):
            assert np.array_equal(eng.initial_state(chain).pack(), orc.initial_state(chain))


def test_tune_cutoff_resolution():
    """P:tests/test_engine.cpp:278-285"""
    counts, X, h = small(8)
    for burnin, want in [(2000, 200), (20000, 500), (50, 5)]:
        eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, h),
                          RunConfig(chains=1, burnin=burnin, iterations=10))
        assert eng.config().tune_cutoff == want


@pytest.mark.parametrize("kw", [dict(tune_cutoff=100), dict(thin=0), dict(workers=0),
                                dict(chains=0), dict(iterations=0)])
def test_config_validation(kw):
    """P:tests/test_engine.cpp:263-276"""
    base = dict(chains=1, burnin=100, iterations=100, seed=17)
    base.update(kw)
    with pytest.raises(ConfigError):
        GibbsEngine(CountMatrix(np.zeros((1, 1), np.int64)), ModelSpec(np.ones((1, 1)), np.zeros(1)),
                    RunConfig(**base))


def test_input_validation():
    X = np.array([[1.0, 1.0], [1.0, 1.0]])  # rank deficient
    with pytest.raises(ConfigError, match="full column rank"):
        GibbsEngine(CountMatrix(np.ones((2, 2), np.int64)), ModelSpec(X, np.zeros(2)),
                    RunConfig(chains=1, burnin=10, iterations=10))
    with pytest.raises(ConfigError, match="negative count"):
        GibbsEngine(CountMatrix(-np.ones((2, 1), np.int64)), ModelSpec(np.ones((1, 1)), np.zeros(1)),
                    RunConfig(chains=1, burnin=10, iterations=10))


def test_param_ref_parsing():
    """P:tests/test_streaming.cpp:62-114"""
    assert parse_param_ref("beta[,2]", 5).index == 1
    assert parse_param_ref("theta[1]", 5).family == "theta"
    assert parse_param_ref("sigma[5]", 5).index == 4
    for bad in ("bogus", "beta[2]", "beta[,0]", "beta[,6]", "theta[0]", "theta[6]",
                "theta[x]", "gamma[1]", "sigma"):
        with pytest.raises(ConfigError):
            parse_param_ref(bad, 5)
    assert heterosis_contrast().per_gene


def test_shard_bounds_are_leaf_aligned_and_cover():
    lib = _abi.load_library()
    for G in (1, 1000, 1024, 39656, 1_000_000, 317248):
        for world in (1, 2, 4, 8):
            prev = 0
            for r in range(world):
                lo, hi = c_long(), c_long()
                assert lib.cmc_shard_bounds(G, r, world, byref(lo), byref(hi)) == 0
                assert lo.value == prev and lo.value % 1024 == 0 or lo.value == G
                assert hi.value >= lo.value
                prev = hi.value
            assert prev == G


def test_simulate_is_deterministic_and_shaped():
    a = small(100, 16, 7)[0]
    b = small(100, 16, 7)[0]
    c = small(100, 16, 8)[0]
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    assert a.dtype == np.int64 and a.min() >= 0 and a.shape == (100, 16)
    # log-mean near theta_1 = 2.5 on average over genes
    assert 1.5 < np.log(a.mean(axis=1) + 1).mean() < 3.5


def test_sample_count_beyond_gene_kernel_shared_memory():
    """The gene kernel keeps lp (N doubles per gene) in shared memory: a
    clear ConfigError at create, not a launch failure later."""
    from paper_1606_06659_b200 import builtin_design
    X = builtin_design("heterosis16x5", 240)
    counts = np.ones((8, 240), np.int64)
    with pytest.raises(ConfigError, match="at most 222 samples"):
        GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(240)),
                    RunConfig(chains=1, burnin=10, iterations=10))
    from helpers import two_col_design
    for N, fits in ((222, True), (223, False)):
        X = two_col_design(N)
        make = lambda: GibbsEngine(CountMatrix(np.ones((8, N), np.int64)),  # noqa: E731
                                   ModelSpec(X, np.zeros(N)),
                                   RunConfig(chains=1, burnin=10, iterations=10))
        if fits:
            make()
        else:
            with pytest.raises(ConfigError, match="at most 222 samples"):
                make()


@pytest.mark.parametrize("G,N,seed,nu,tau,theta", [
    (2000, 16, 1, 8.0, 0.7, [2.5, .2, .2, 0.0, .1]),    # the bench data (Paschold-shaped)
    (400, 64, 1, 8.0, 0.7, [2.5, .2, .2, 0.0, .1]),     # config 5's N = 64 tiling
    (300, 16, 9, 3.0, 0.5, [6.0, .5, .2, 0.0, .1]),     # large means: PTRD branch only
    (300, 16, 4, 8.0, 0.7, [0.5, .2, .2, 0.0, .1]),     # small means: product branch
])
def test_simulate_equals_reference_generate(ref, G, N, seed, nu, tau, theta):
    """cmc_simulate draws the reference's generate() (P:src/simulate.cpp:
    28-90) bit for bit: same Philox site per gene, same normal/gamma draw
    order, and std::poisson_distribution<long long> over the same stream, so
    the bench's two arms consume identical arrays."""
    import oracle
    sigma = [.4, .25, .25, .15, .2]
    X = builtin_design("heterosis16x5", N)
    ours = generate(SimSpec(G=G, N=N, X=X, nu=nu, tau=tau, theta=theta, sigma=sigma,
                            seed=seed)).counts
    theirs, Xr = oracle.ref_generate(G, N, nu, tau, theta, sigma, seed)
    assert np.array_equal(X, Xr)
    assert np.array_equal(ours, theirs)


def test_simulate_overflow_error_matches_reference(ref):
    import oracle
    X = builtin_design("heterosis16x5", 16)
    kw = dict(nu=8.0, tau=0.7, theta=[800.0, 0, 0, 0, 0], sigma=[0.0] * 5, seed=1)
    with pytest.raises(ConfigError) as ours:
        generate(SimSpec(G=3, N=16, X=X, **kw))
    with pytest.raises(oracle.ConfigErr) as theirs:
        oracle.ref_generate(3, 16, kw["nu"], kw["tau"], kw["theta"], kw["sigma"], 1)
    assert str(ours.value) == str(theirs.value)
