"""GPU: the gene-sharded path at world > 1 on one B200.  W engines of this
process join an in-process loopback group (cmc_engine_shard_loopback) and
run as ranks 0..W-1, one host thread each.  The all-gather of the leaf
partials becomes event-ordered device copies between the engines, so no
kernel waits on another.  Everything else is the multi-GPU code path:
  * leaf-aligned shard bounds;
  * RNG sites offset by the shard's first gene;
  * [world][C][Q][lpr] partial sections;
  * the standalone hyper kernels.
Every rank's genes and every rank's hyperparameters must be bit-identical to
one unsharded engine (and so to the reference: the fused path is pinned
against the oracle elsewhere)."""
import threading

import numpy as np
import pytest

from paper_1606_06659_b200 import (CountMatrix, GibbsEngine, LoopbackGroup, ModelSpec,
                                   RunConfig, heterosis_contrast)

from helpers import heterosis

pytestmark = pytest.mark.gpu


def _run_ranks(counts, X, h, cfg, world, contrasts=(), priors=None):
    group = LoopbackGroup(world)
    engines = []
    for r in range(world):
        e = GibbsEngine(CountMatrix(counts), ModelSpec(X, h, priors=priors) if priors
                        else ModelSpec(X, h), cfg, contrasts=list(contrasts))
        e.shard_loopback(r, group)
        engines.append(e)
    outs, errs = [None] * world, []

    def work(r):
        try:
            outs[r] = engines[r].run()
        except Exception as ex:  # surfaced below
            errs.append(ex)

    # daemon threads: a hung rank cannot keep the test process alive
    threads = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in threads), "loopback ranks did not finish"
    assert not errs, errs
    return engines, outs


def _same(a, b, what):
    assert np.array_equal(a, b), what


def _check(fused, engines, outs, chains, L):
    for r, (e, out) in enumerate(zip(engines, outs)):
        lo, hi = e.shard_range
        for c in range(chains):
            a, b = fused[c], out[c]
            tag = f"rank {r} chain {c}"
            # genes of this shard
            for name in ("eps", "gamma", "beta"):
                _same(getattr(a.final_state, name)[lo:hi], getattr(b.final_state, name)[lo:hi],
                      f"{tag} final {name}")
            if a.final_state.xi is not None:
                _same(a.final_state.xi[lo:hi], b.final_state.xi[lo:hi], f"{tag} final xi")
            for acc in ("beta_acc", "gamma_acc", "eps_acc") + (("xi_acc",) if a.xi_acc else ()):
                for k in ("mean", "meansq"):
                    _same(getattr(getattr(a, acc), k)[lo:hi], getattr(getattr(b, acc), k)[lo:hi],
                          f"{tag} {acc}.{k}")
            for ca, cb in zip(a.contrasts, b.contrasts):
                if ca.prob.shape[0] > 1:
                    _same(ca.prob[lo:hi], cb.prob[lo:hi], f"{tag} contrast prob")
                else:
                    _same(ca.prob, cb.prob, f"{tag} contrast prob")
            # hyperparameters: every rank holds the full values
            for name in ("theta", "sigma"):
                _same(getattr(a.final_state, name), getattr(b.final_state, name), f"{tag} {name}")
            assert a.final_state.nu == b.final_state.nu and a.final_state.tau == b.final_state.tau
            for acc in ("nu_acc", "tau_acc", "theta_acc", "sigma_acc"):
                for k in ("mean", "meansq"):
                    _same(getattr(getattr(a, acc), k), getattr(getattr(b, acc), k), f"{tag} {acc}")
            _same(a.samples[:2 + 2 * L], b.samples[:2 + 2 * L], f"{tag} hyper samples")
            # saved genes inside the shard
            for k, g in enumerate(a.saved_genes):
                if lo <= g < hi:
                    c0 = 2 + 2 * L + k * (L + 1)
                    _same(a.samples[c0:c0 + L + 1], b.samples[c0:c0 + L + 1], f"{tag} gene {g}")
    # clamp events are counted per shard
    for c in range(chains):
        assert sum(o[c].clamp_events for o in outs) == fused[c].clamp_events


@pytest.mark.parametrize("G,world", [(2500, 2), (5000, 3), (7000, 4)])
def test_sharded_run_equals_single_engine(G, world):
    counts, X, h = heterosis(G, seed=6)
    cfg = RunConfig(chains=2, burnin=25, iterations=30, thin=5, seed=8, save_genes=12)
    cons = [heterosis_contrast()]
    fused = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg, contrasts=cons).run()
    engines, outs = _run_ranks(counts, X, h, cfg, world, contrasts=cons)
    assert [e.shard_range for e in engines][-1][1] == G
    _check(fused, engines, outs, 2, X.shape[1])


def test_sharded_run_with_xi_prior_and_hyper_contrast():
    """ξ columns add Q sections (2 + 2L); a contrast on a hyperparameter and a
    gene parameter needs the hyper step's values inside each shard."""
    from paper_1606_06659_b200 import ContrastSpec, ContrastTerm, ParamRef, PriorConfig
    counts, X, h = heterosis(2100, seed=9)
    cfg = RunConfig(chains=3, burnin=20, iterations=20, thin=4, seed=2, save_genes=6)
    pri = PriorConfig(beta_prior=["normal", "laplace", "t", "horseshoe", "normal"], t_df=3.0)
    cons = [ContrastSpec(id="b1_gt_theta1",
                         terms=[ContrastTerm(coeffs=[(ParamRef("beta_col", 1), 1.0),
                                                     (ParamRef("theta", 1), -1.0)],
                                             threshold=0.0)])]
    fused = GibbsEngine(CountMatrix(counts), ModelSpec(X, h, priors=pri), cfg,
                        contrasts=cons).run()
    engines, outs = _run_ranks(counts, X, h, cfg, 2, contrasts=cons, priors=pri)
    _check(fused, engines, outs, 3, X.shape[1])


def test_rank_without_genes_is_a_config_error():
    """Sections are ceil(leaves / world) leaves each (the all-gather moves
    equal counts), so 4 leaves over 3 ranks leave rank 2 empty: refused at
    shard time, as cmc_engine_shard does."""
    from paper_1606_06659_b200 import ConfigError
    counts, X, h = heterosis(3100, seed=6)
    cfg = RunConfig(chains=1, burnin=5, iterations=5, thin=5, seed=8)
    group = LoopbackGroup(3)
    e = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg)
    with pytest.raises(ConfigError):
        e.shard_loopback(2, group)


def test_sharded_job_results_files_equal_single_engine(tmp_path):
    """The multi-GPU user flow: every rank runs its shard, the outputs are
    merged (shards.merge_shard_outputs, what gather_shard_outputs does on
    rank 0), loaded into an unsharded engine of the full problem
    (load_outputs), which writes the reference's result files.  Every file
    equals the one a single unsharded engine writes; run_report.json
    differs only in its device-time field."""
    import json
    from paper_1606_06659_b200.shards import merge_shard_outputs
    counts, X, h = heterosis(5000, seed=12)
    cfg = RunConfig(chains=3, burnin=20, iterations=40, thin=5, seed=4, save_genes=10)
    cons = [heterosis_contrast()]
    single = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg, contrasts=cons)
    single.run()
    single.write_results(str(tmp_path / "single"), wall_seconds=1.5)
    engines, outs = _run_ranks(counts, X, h, cfg, 3, contrasts=cons)
    merged = merge_shard_outputs(outs, [e.shard_range for e in engines])
    res = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg, contrasts=cons)
    res.load_outputs(merged)
    res.write_results(str(tmp_path / "sharded"), wall_seconds=1.5)
    a, b = tmp_path / "single", tmp_path / "sharded"
    files = sorted(p.relative_to(a) for p in a.rglob("*") if p.is_file())
    assert files == sorted(p.relative_to(b) for p in b.rglob("*") if p.is_file())
    for f in files:
        if f.name == "run_report.json":
            def strip(j):  # device seconds differ run to run
                if isinstance(j, dict):
                    return {k: strip(v) for k, v in j.items() if k != "step_seconds"}
                return [strip(v) for v in j] if isinstance(j, list) else j
            assert strip(json.loads((a / f).read_text())) == strip(json.loads((b / f).read_text()))
        else:
            assert (a / f).read_bytes() == (b / f).read_bytes(), f
    da, db = single.diagnostics(), res.diagnostics()
    for k in ("rhat", "mean", "sd", "ci_lo", "ci_hi", "ess"):
        assert np.array_equal(getattr(da, k), getattr(db, k), equal_nan=True), k
