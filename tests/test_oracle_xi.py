"""ξ-augmented β priors: the oracle restatement.

The reference has no ξ sampler, so parity is UNPINNED: these tests pin the
restatement itself:
  * the log full conditionals against their closed forms;
  * the slice sampler on each conditional against the exact law, a KS test;
  * the engine-level bookkeeping (layouts, ξ > 0, normal columns untouched).
The GPU is then held bit-for-bit to this oracle (tests/test_gpu_xi.py)."""
import math
from ctypes import POINTER, c_double

import numpy as np
import pytest
from scipy import integrate, stats

import oracle
from paper_1606_06659_b200 import _abi

from helpers import heterosis

L_ = oracle.load_oracle()
LAPLACE, T, HORSESHOE = 1, 2, 3


def test_log_conditionals_closed_forms():
    for xi in (1e-3, 0.37, 1.0, 2.5, 40.0):
        for q in (0.0, 0.7, 12.0):
            assert L_.orc_log_fc_xi(LAPLACE, xi, q, 0.0) == \
                -0.5 * math.log(xi) - q / xi - 0.5 * xi
            assert L_.orc_log_fc_xi(T, xi, q, 3.0) == \
                -(0.5 * 3.0 + 1.5) * math.log(xi) - (q + 0.5 * 3.0) / xi
            assert L_.orc_log_fc_xi(HORSESHOE, xi, q, 0.0) == \
                -math.log(xi * (1.0 + xi)) - q / xi
            assert abs(L_.orc_log_fc_xi(HORSESHOE, xi, q, 0.0) -
                       (-math.log(xi) - q / xi - math.log1p(xi))) < 1e-13 * (1 + q / xi)
    for xi in (1e151, 1e200):   # x (1 + x) would overflow: the two-log form
        assert L_.orc_log_fc_xi(HORSESHOE, xi, 0.5, 0.0) == \
            -math.log(xi) - 0.5 / xi - math.log1p(xi)
    for fam in (LAPLACE, T, HORSESHOE):
        assert L_.orc_log_fc_xi(fam, 0.0, 0.7, 3.0) == -math.inf
        assert L_.orc_log_fc_xi(fam, -1.0, 0.7, 3.0) == -math.inf


def _chain(density, n=20000, burnin=200, seed=5):
    out = np.zeros(n)
    rc = L_.orc_slice_chain(density, 1.0, n, burnin, 1.0, seed,
                            out.ctypes.data_as(POINTER(c_double)))
    assert rc == 0
    return out[::5]


def test_t_conditional_is_inverse_gamma():
    # q = 0.7, k = 3: xi | . ~ IG((k+1)/2, q + k/2) = IG(2, 2.2)
    x = _chain(4)
    assert stats.kstest(x, stats.invgamma(a=2.0, scale=2.2).cdf).pvalue > 0.01


def test_laplace_conditional_is_gig():
    # xi^(-1/2) exp(-(q/xi + xi/2)): GIG(p = 1/2, chi = 2q, psi = 1)
    chi, psi = 1.4, 1.0
    law = stats.geninvgauss(p=0.5, b=math.sqrt(chi * psi), scale=math.sqrt(chi / psi))
    x = _chain(5, seed=8)
    assert stats.kstest(x, law.cdf).pvalue > 0.01


def test_horseshoe_conditional_numerical_cdf():
    q = 0.7
    dens = lambda v: math.exp(-math.log(v) - q / v - math.log1p(v))  # noqa: E731
    Z = integrate.quad(dens, 0, np.inf, limit=200)[0]
    x = _chain(6, seed=13)
    grid = np.quantile(x, [0.05, 0.25, 0.5, 0.75, 0.95])
    for g, p in zip(grid, [0.05, 0.25, 0.5, 0.75, 0.95]):
        F = integrate.quad(dens, 0, g, limit=200)[0] / Z
        assert F == pytest.approx(p, abs=0.02)


def _engine(prior, G=60, chains=1, seed=3):
    counts, X, h = heterosis(G, seed=seed)
    cfg = _abi.make_config(chains=chains, burnin=20, iterations=30, thin=5, seed=seed,
                           save_genes=3)
    return oracle.OracleEngine(counts, X, h, cfg,
                               priors={"beta_prior": prior, "t_df": 3.0})


@pytest.mark.parametrize("prior", [["laplace"], ["t"], ["horseshoe"],
                                   ["normal", "laplace", "normal", "t", "horseshoe"]])
def test_engine_layout_and_support(prior):
    eng = _engine(prior)
    G, N, L = eng.G, eng.N, eng.L
    S, T_, A = _abi.sizes(G, N, L, True)
    st = eng.initial_state(1)
    assert len(st) == S and np.all(st[S - G * L:] == 1.0)
    out = eng.run_chain(0)
    xi = out["final"][S - G * L:].reshape(G, L)
    codes = [_abi.PRIORS[p] for p in (prior * L if len(prior) == 1 else prior)]
    for l, c in enumerate(codes):
        if c == 0:
            assert np.all(xi[:, l] == 1.0)          # normal columns never move
        else:
            assert np.all(xi[:, l] > 0) and len(np.unique(xi[:, l])) > G // 2
    # xi accumulators close the accumulator block
    assert len(out["mean"]) == A
    assert np.allclose(out["mean"][A - G * L:].reshape(G, L)[:, [l for l, c in
                       enumerate(codes) if c == 0]], 1.0)


def test_all_normal_prior_is_the_reference_model():
    """beta_prior all 'normal' takes the reference path: same bits as no prior."""
    counts, X, h = heterosis(40, seed=1)
    cfg = _abi.make_config(chains=1, burnin=10, iterations=10, thin=5, seed=9)
    a = oracle.OracleEngine(counts, X, h, cfg).run_chain(0)
    b = oracle.OracleEngine(counts, X, h, cfg, priors={"beta_prior": ["normal"]}).run_chain(0)
    assert np.array_equal(a["final"], b["final"]) and np.array_equal(a["mean"], b["mean"])


def test_bad_prior_config():
    counts, X, h = heterosis(10, seed=1)
    cfg = _abi.make_config(chains=1, burnin=10, iterations=10)
    with pytest.raises(oracle.ConfigErr, match="t prior needs positive"):
        oracle.OracleEngine(counts, X, h, cfg, priors={"beta_prior": ["t"], "t_df": 0.0})
    with pytest.raises(oracle.ConfigErr, match="beta prior must be"):
        oracle.OracleEngine(counts, X, h, cfg, priors={"beta_prior": [7]})


def test_laplace_shrinks_harder_than_normal_near_zero():
    """Posterior sanity on simulated data: with a Laplace prior the small
    effects (column 4, true theta 0) are pulled closer to theta than the
    normal prior pulls them."""
    counts, X, h = heterosis(200, seed=4)
    cfg = _abi.make_config(chains=1, burnin=200, iterations=300, thin=10, seed=2)
    S, _, _ = _abi.sizes(200, counts.shape[1], X.shape[1])
    nrm = oracle.OracleEngine(counts, X, h, cfg).run_chain(0)
    lap = oracle.OracleEngine(counts, X, h, cfg,
                              priors={"beta_prior": ["laplace"]}).run_chain(0)
    L = X.shape[1]
    b0 = 2 + 2 * L
    bn = nrm["mean"][b0:b0 + 200 * L].reshape(200, L)[:, 3]
    bl = lap["mean"][b0:b0 + 200 * L].reshape(200, L)[:, 3]
    assert np.median(np.abs(bl - np.median(bl))) < np.median(np.abs(bn - np.median(bn))) * 1.05
