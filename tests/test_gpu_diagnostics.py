"""GPU: post-run diagnostics computed on the device from the resident
accumulators equal the reference's build_diagnostics numerics
(gelman_rhat, pool_moments + credible_interval, effective_sample_size;
P:src/io.cpp:507-569, P:src/diagnostics.cpp) run on the reference's own
ChainOutputs (oracle/_ref).  R-hat, pooled moments and ESS are bit-identical
wherever the accumulators are (every row but theta); theta rows and the
intervals (AS241 z through log) agree to 1e-12."""
import numpy as np
import pytest

import oracle
from paper_1606_06659_b200 import (CountMatrix, GibbsEngine, ModelSpec, RunConfig,
                                   heterosis_contrast)

from helpers import heterosis, mismatch

pytestmark = pytest.mark.gpu


@pytest.mark.usefixtures("ref")
@pytest.mark.parametrize("chains,thin", [(2, 5), (4, 10)])
def test_device_diagnostics_match_reference(chains, thin):
    counts, X, h = heterosis(150, seed=12)
    cfg = RunConfig(chains=chains, burnin=30, iterations=60, thin=thin, seed=21, save_genes=7)
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg)
    d = eng.diagnostics()
    ref = oracle.RefEngine(counts, X, h, cfg.to_c()).diagnostics(eng.n_cols)
    G, L = 150, 5
    R = 2 + 2 * L + G * (L + 1)
    theta = np.zeros(R, bool)
    theta[2:2 + L] = True
    for k in ("rhat", "mean", "sd"):
        got = getattr(d, k)
        assert not len(mismatch(got[~theta], ref[k][~theta])), k
        np.testing.assert_allclose(got[theta], ref[k][theta], rtol=1e-12)
    np.testing.assert_allclose(d.ci_lo, ref["lo"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(d.ci_hi, ref["hi"], rtol=1e-12, atol=1e-15)
    assert np.array_equal(d.degenerate, (ref["flags"] & 1) != 0)
    assert np.array_equal(d.passed, (ref["flags"] & 2) != 0)
    # ESS: hyper columns in sample order, then saved genes
    sv = eng.saved_genes()
    cols = list(range(2 + 2 * L))
    rows = list(range(2 + 2 * L))
    for k, g in enumerate(sv):
        for l in range(L):
            cols.append(2 + 2 * L + k * (L + 1) + l)
            rows.append(2 + 2 * L + g * L + l)
        cols.append(2 + 2 * L + k * (L + 1) + L)
        rows.append(2 + 2 * L + G * L + g)
    for c, r in zip(cols, rows):
        st = {0: "ok", 1: "undefined", 2: "degenerate"}[int(ref["ess_status"][c])]
        assert d.ess_status[r] == st
        if st == "ok":
            if 2 <= r < 2 + L:
                assert d.ess[r] == pytest.approx(ref["ess"][c], rel=1e-12)
            else:
                assert d.ess[r] == ref["ess"][c]
    assert d.ess_status[2 + 2 * L + [g for g in range(G) if g not in set(sv)][0] * L] == \
        "not-retained"
    assert d.names[0] == "nu" and d.names[2 + 2 * L] == "beta[1,1]" and d.names[-1] == "gamma[150]"


def test_diagnostics_need_two_chains():
    counts, X, h = heterosis(64, seed=3)
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, h),
                      RunConfig(chains=1, burnin=10, iterations=10, seed=1))
    from paper_1606_06659_b200 import ConfigError
    with pytest.raises(ConfigError, match="2 chains"):
        eng.diagnostics()


def test_paschold_shape_diagnostics_pipeline():
    """4 chains x (200 + 400) sweeps at G = 39,656 (BASELINE configs[1]):
    the device diagnostics cover all 2 + 2L + G(L+1) rows with finite,
    ordered values (short chains need not have converged: the reference's
    own mode-agreement criterion runs 2000 + 6000 sweeps)."""
    counts, X, h = heterosis(39656, seed=1)
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, h),
                      RunConfig(chains=4, burnin=200, iterations=400, thin=20, seed=7),
                      contrasts=[heterosis_contrast()])
    d = eng.diagnostics()
    assert len(d.rhat) == 2 + 10 + 39656 * 6
    assert np.all(np.isfinite(d.rhat)) and np.all(d.rhat > 0.5)
    assert np.all(d.ci_lo <= d.mean) and np.all(d.mean <= d.ci_hi)
    assert not d.degenerate.any()
    assert sum(s == "ok" for s in d.ess_status) == eng.n_cols


@pytest.mark.usefixtures("ref")
def test_long_thinned_run_ess_matches_reference():
    """20,000 retained rows per column (thin 1): the ESS kernel computes lags
    in batches and stops at the Geyer cutoff like the reference's lazy
    avg_autocov, with the same bits."""
    counts, X, h = heterosis(30, seed=5)
    cfg = RunConfig(chains=2, burnin=100, iterations=20000, thin=1, seed=8, save_genes=2)
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg)
    d = eng.diagnostics()
    ref = oracle.RefEngine(counts, X, h, cfg.to_c()).diagnostics(eng.n_cols)
    L = 5
    hyper = list(range(2 + 2 * L))
    for c in hyper:
        st = {0: "ok", 1: "undefined", 2: "degenerate"}[int(ref["ess_status"][c])]
        assert d.ess_status[c] == st
        if st == "ok":
            if 2 <= c < 2 + L:
                assert d.ess[c] == pytest.approx(ref["ess"][c], rel=1e-10)
            else:
                assert d.ess[c] == ref["ess"][c], c
