"""GPU parity: the CUDA sweep against the oracle (countmc_oracle.c, itself
pinned bit-for-bit to the compiled reference) on identical inputs.

Tolerance (BASELINE.json north_star: 1e-12 relative for a single sweep):
every slice-sampled value (eps, gamma, beta, nu, tau, sigma) and all slice
widths must be BIT-IDENTICAL — their values depend only on the shared
Philox uniforms and the outcomes of comparisons (SURVEY.md §7 hard part 1);
theta (AS241 tail uses log) and conjugate-direct draws (pow/log inside
Marsaglia-Tsang) may differ in the last bits, bounded by REL_TOL.
"""
import numpy as np
import pytest

import oracle
from paper_1606_06659_b200 import _abi
from paper_1606_06659_b200._abi import sizes

from helpers import (HETEROSIS, Product, advance, heterosis, mismatch, packed_start,
                     simulated, tiny)

pytestmark = pytest.mark.gpu
REL_TOL = 1e-12


def theta_slice(G, N, L):
    o = G * N + G + G * L
    return slice(o, o + L)


def assert_state_parity(a, b, G, N, L, what=""):
    bad = mismatch(a, b)
    th = theta_slice(G, N, L)
    th_idx = set(range(th.start, th.stop))
    rest = [i for i in bad if i not in th_idx]
    assert not rest, f"{what}: non-bitwise state entries {rest[:10]}"
    np.testing.assert_allclose(a[th], b[th], rtol=REL_TOL, atol=0)


def run_pair(counts, X, h, cfg, chain, sweeps, start=None, priors=None):
    orc = oracle.OracleEngine(counts, X, h, cfg, priors=priors)
    gpu = Product(counts, X, h, cfg, priors=priors)
    st, tw, ta = packed_start(orc, chain, cfg.w_init)
    m0 = 1
    if start:
        advance(orc, st, tw, ta, chain, 1, start)
        m0 = start
    g_st, g_tw, g_ta = st.copy(), tw.copy(), ta.copy()
    G, N = counts.shape
    L = X.shape[1]
    for m in range(m0, m0 + sweeps):
        c1 = orc.iterate(st, tw, ta, chain, m)
        c2 = gpu.iterate(g_st, g_tw, g_ta, chain, m)
        assert c1 == c2, f"clamp count m={m}: {c1} vs {c2}"
        assert_state_parity(g_st, st, G, N, L, f"m={m}")
        assert not len(mismatch(g_tw, tw)), f"w differs at m={m}"
        assert not len(mismatch(g_ta, ta)), f"w_aux differs at m={m}"
    return st


def test_tiny_sweeps_bitwise():
    counts, X, h = tiny()
    cfg = _abi.make_config(chains=1, burnin=100, iterations=900, thin=20, seed=17,
                           tune_cutoff=10, save_genes=8)
    run_pair(counts, X, h, cfg, 0, 40)


def test_two_column_design_sweeps_bitwise():
    counts, X, h = simulated(64, 4, 5)
    cfg = _abi.make_config(chains=1, burnin=40, iterations=60, thin=20, seed=17,
                           tune_cutoff=4, save_genes=8)
    run_pair(counts, X, h, cfg, 0, 60)


@pytest.mark.parametrize("chain", [0, 2])
def test_heterosis_g1000_single_sweep_bitwise(chain):
    counts, X, h = heterosis(1000)
    cfg = _abi.make_config(chains=3, burnin=50, iterations=50, thin=10, seed=3, save_genes=10)
    run_pair(counts, X, h, cfg, chain, 3)
    # steady state after tuning (widths tuned, m > tune_cutoff)
    run_pair(counts, X, h, cfg, chain, 2, start=30)


def test_heterosis_paschold_shape_single_sweep():
    counts, X, h = heterosis(39656, seed=1)
    cfg = _abi.make_config(chains=1, burnin=200, iterations=100, thin=20, seed=7)
    run_pair(counts, X, h, cfg, 0, 1)


def test_run_matches_oracle_run_chain():
    counts, X, h = heterosis(200, seed=8)
    cfg = _abi.make_config(chains=2, burnin=30, iterations=50, thin=5, seed=17, save_genes=12)
    orc = oracle.OracleEngine(counts, X, h, cfg, contrasts=[HETEROSIS])
    gpu = Product(counts, X, h, cfg, contrasts=[HETEROSIS])
    outs = gpu.run()
    G, N, L = 200, 16, 5
    S, _, A = sizes(G, N, L)
    th = slice(2, 2 + L)  # theta accumulators
    for c in range(2):
        ref = orc.run_chain(c)
        got = outs[c]
        assert got["count"][0] == ref["count"][0] == 50
        assert got["clamps"][0] == ref["clamps"][0]
        assert_state_parity(got["final"], ref["final"], G, N, L, f"chain {c} final")
        for k in ("mean", "meansq"):
            bad = [i for i in mismatch(got[k], ref[k]) if not (th.start <= i < th.stop)]
            assert not bad, (c, k, bad[:10])
            np.testing.assert_allclose(got[k], ref[k], rtol=REL_TOL)
        np.testing.assert_array_equal(got["iters"], ref["iters"])
        np.testing.assert_allclose(got["samples"], ref["samples"], rtol=REL_TOL)
        np.testing.assert_allclose(got["prob"], ref["prob"], rtol=REL_TOL)


def test_conjugate_direct_mode_within_tolerance():
    counts, X, h = simulated(20, 4, 6)
    cfg = _abi.make_config(chains=1, burnin=30, iterations=50, thin=20, seed=17,
                           tune_cutoff=3, sampler_mode=_abi.CMC_CONJUGATE_DIRECT)
    orc = oracle.OracleEngine(counts, X, h, cfg)
    gpu = Product(counts, X, h, cfg)
    st, tw, ta = packed_start(orc, 0)
    g = (st.copy(), tw.copy(), ta.copy())
    orc.iterate(st, tw, ta, 0, 1)
    gpu.iterate(*g, 0, 1)
    np.testing.assert_allclose(g[0], st, rtol=1e-12)


def test_stall_reports_step_and_coordinates():
    counts, X, h = simulated(8, 4, 11)
    cfg = _abi.make_config(chains=1, burnin=50, iterations=50, thin=20, seed=17,
                           tune_cutoff=5, save_genes=8, max_shrink=1)
    gpu = Product(counts, X, h, cfg)
    with pytest.raises(oracle.StallError) as ei:
        gpu.run()
    e = ei.value
    assert e.step
    assert e.iteration >= 1
    assert e.step in str(e)
    # same first stall as the sequential reference sweep
    orc = oracle.OracleEngine(counts, X, h, cfg)
    with pytest.raises(oracle.StallError) as eo:
        orc.run_chain(0)
    assert (e.step, e.index1, e.index2, e.iteration) == \
        (eo.value.step, eo.value.index1, eo.value.index2, eo.value.iteration)
    assert e.x0 == eo.value.x0 and e.width == eo.value.width
