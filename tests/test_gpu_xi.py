"""GPU: ξ-augmented β priors (BASELINE configs 2-3)
against the oracle restatement (tests/test_oracle_xi.py pins that oracle to
the closed-form conditionals).  The reference has no ξ sampler, so this is
parity with OUR restatement, not with the reference: "parity unpinned".

Bar: as for the reference model -- every slice-sampled value (now including
ξ and its widths) bit-identical; θ within 1e-12 relative."""
import numpy as np
import pytest

import oracle
from paper_1606_06659_b200 import (CountMatrix, GibbsEngine, ModelSpec, PriorConfig,
                                   RunConfig, _abi, heterosis_contrast)
from paper_1606_06659_b200._abi import sizes

from helpers import Product, advance, heterosis, mismatch, packed_start

pytestmark = pytest.mark.gpu
REL_TOL = 1e-12
PRIORS = [["laplace"], ["t"], ["horseshoe"], ["normal", "laplace", "t", "horseshoe", "laplace"]]


def _pair(prior, G=300, chains=2, burnin=40, seed=5, t_df=3.0):
    counts, X, h = heterosis(G, seed=seed)
    cfg = _abi.make_config(chains=chains, burnin=burnin, iterations=40, thin=10, seed=seed,
                           save_genes=5)
    pr = {"beta_prior": prior, "t_df": t_df}
    return (oracle.OracleEngine(counts, X, h, cfg, priors=pr),
            Product(counts, X, h, cfg, priors=pr), counts.shape[0], counts.shape[1], X.shape[1])


def _state_parity(a, b, G, N, L, what):
    th0 = G * N + G + G * L
    bad = [i for i in mismatch(a, b) if not th0 <= i < th0 + L]
    assert not bad, f"{what}: non-bitwise entries {bad[:10]}"
    np.testing.assert_allclose(a[th0:th0 + L], b[th0:th0 + L], rtol=REL_TOL, atol=0)


@pytest.mark.parametrize("prior", PRIORS)
@pytest.mark.parametrize("chain", [0, 1])
def test_sweeps_bitwise_vs_oracle(prior, chain):
    orc, gpu, G, N, L = _pair(prior)
    st, tw, ta = packed_start(orc, chain)
    assert len(st) == sizes(G, N, L, True)[0]
    g = [st.copy(), tw.copy(), ta.copy()]
    for m in range(1, 8):   # burn-in sweeps: widths tune, xi moves off 1
        c1 = orc.iterate(st, tw, ta, chain, m)
        c2 = gpu.iterate(*g, chain, m)
        assert c1 == c2
        _state_parity(g[0], st, G, N, L, f"m={m}")
        assert not len(mismatch(g[1], tw)) and not len(mismatch(g[2], ta))
    xi = st[-G * L:].reshape(G, L)
    assert np.all(xi > 0)


@pytest.mark.parametrize("prior", [["laplace"], ["horseshoe"]])
def test_steady_state_sweeps_bitwise(prior):
    orc, gpu, G, N, L = _pair(prior, G=1000, burnin=30)
    st, tw, ta = packed_start(orc, 0)
    advance(orc, st, tw, ta, 0, 1, 35)      # tuned, past burn-in
    g = [st.copy(), tw.copy(), ta.copy()]
    for m in range(35, 38):
        assert orc.iterate(st, tw, ta, 0, m) == gpu.iterate(*g, 0, m)
        _state_parity(g[0], st, G, N, L, f"m={m}")


@pytest.mark.parametrize("prior", [["t"], ["normal", "laplace", "t", "horseshoe", "laplace"]])
def test_run_outputs_match_oracle(prior):
    """run(): accumulators including the xi block, thinned samples, final
    states, for every chain (batched on the device)."""
    orc, gpu, G, N, L = _pair(prior, G=200, chains=3, burnin=20)
    outs = gpu.run()
    for c in range(3):
        o = orc.run_chain(c)
        _state_parity(outs[c]["final"], o["final"], G, N, L, f"chain {c}")
        A = sizes(G, N, L, True)[2]
        skip = set(range(2, 2 + L))  # theta accumulators: 1e-12 (theta draws)
        for k in ("mean", "meansq"):
            bad = [i for i in mismatch(outs[c][k], o[k]) if i not in skip]
            assert not bad, (c, k, bad[:5])
            np.testing.assert_allclose(outs[c][k][2:2 + L], o[k][2:2 + L], rtol=1e-10)
        assert len(outs[c]["mean"]) == A
        xi_mean = outs[c]["mean"][A - G * L:].reshape(G, L)
        codes = [_abi.PRIORS[p] for p in (prior * L if len(prior) == 1 else prior)]
        for l, code in enumerate(codes):
            if code == 0:
                assert np.all(xi_mean[:, l] == 1.0)
            else:
                assert np.all(xi_mean[:, l] > 0)


def test_xi_stall_reported_like_oracle():
    counts, X, h = heterosis(16, seed=2)
    cfg = _abi.make_config(chains=1, burnin=20, iterations=20, thin=10, seed=4,
                           max_shrink=1, save_genes=2)
    pr = {"beta_prior": ["horseshoe"]}
    with pytest.raises(oracle.StallError) as eo:
        oracle.OracleEngine(counts, X, h, cfg, priors=pr).run_chain(0)
    with pytest.raises(oracle.StallError) as eg:
        Product(counts, X, h, cfg, priors=pr).run()
    a, b = eg.value, eo.value
    assert (a.step, a.index1, a.index2, a.iteration) == (b.step, b.index1, b.index2, b.iteration)
    assert a.x0 == b.x0 and a.width == b.width


def test_python_api_with_laplace_prior():
    counts, X, h = heterosis(500, seed=6)
    spec = ModelSpec(X, h, PriorConfig(beta_prior=["laplace"]))
    eng = GibbsEngine(CountMatrix(counts), spec,
                      RunConfig(chains=2, burnin=50, iterations=100, thin=10, seed=3),
                      contrasts=[heterosis_contrast()])
    outs = eng.run()
    assert outs[0].xi_acc is not None and outs[0].xi_acc.mean.shape == (500, 5)
    assert np.all(outs[0].xi_acc.mean > 0)
    assert outs[0].final_state.xi.shape == (500, 5)
    d = eng.diagnostics()
    assert np.all(np.isfinite(d.rhat))
    st, tu = eng.initial_state(1), eng.tuning_state()
    eng.iterate(st, tu, 1, 1)
    assert st.xi is not None and np.all(st.xi > 0)


@pytest.mark.parametrize("trips", ["0", "1", "3"])
def test_parked_horseshoe_steps_resume_bitwise(trips, monkeypatch):
    """xi_park_kernel: with a small first-pass trip budget nearly every
    horseshoe lane parks its slice state and Philox queue in shared memory
    and is resumed by another thread; the sweeps stay bit-identical to the
    oracle (burn-in and steady state, a mixed design included)."""
    monkeypatch.setenv("CMC_XI_TRIPS", trips)
    for prior in (["horseshoe"], ["normal", "laplace", "t", "horseshoe", "laplace"]):
        orc, gpu, G, N, L = _pair(prior, G=700, burnin=20)
        st, tw, ta = packed_start(orc, 1)
        g = [st.copy(), tw.copy(), ta.copy()]
        for m in list(range(1, 6)) + [25, 26]:
            assert orc.iterate(st, tw, ta, 1, m) == gpu.iterate(*g, 1, m)
            _state_parity(g[0], st, G, N, L, f"{prior} trips={trips} m={m}")
            assert not len(mismatch(g[1], tw)) and not len(mismatch(g[2], ta))
