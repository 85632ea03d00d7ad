"""GPU parity at BASELINE.json's large configs, at their stated sizes.

* configs[3]: G = 1,000,000, N = 16, L = 5 (heterosis16x5);
* configs[4]: G = 200,000, N = 64, L = 5 (heterosis16x5 tiled to 64 samples:
  64 KB of gene-kernel shared memory per block, the opt-in path).

Each runs the sweep P:src/engine.cpp:161-370 against the compiled reference
itself (oracle/_ref, its own GibbsEngine::iterate on all host threads: the
reference is bitwise independent of its worker count,
P:tests/test_engine.cpp:101-129): two burn-in sweeps from chain 1's jittered
start (tuning active, widths from w_init), then two monitored-phase sweeps
after tune_cutoff and burn-in (widths frozen).  Bar as everywhere: every
slice-sampled value and every width bit-identical, theta within 1e-12.

Also at G = 1M: the gene-sharded path at world 8 (the 8-GPU partition, run
as eight in-process loopback ranks on this GPU) against one unsharded engine,
bit for bit, and the cross-rank stall contract (every rank raises the same
SamplerStallError as one engine)."""
import os
import threading

import numpy as np
import pytest

import oracle
from paper_1606_06659_b200 import (CountMatrix, GibbsEngine, LoopbackGroup, ModelSpec,
                                   RunConfig, SamplerStallError, _abi, heterosis_contrast)
from paper_1606_06659_b200._abi import sizes

from helpers import Product, heterosis, mismatch

pytestmark = pytest.mark.gpu
REL_TOL = 1e-12


def _threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _compare(g, r, G, N, L, what):
    st, tw, ta = g
    rst, rtw, rta = r
    th0 = G * N + G + G * L
    bad = [i for i in mismatch(st, rst) if not th0 <= i < th0 + L]
    assert not bad, f"{what}: state differs at {bad[:8]}"
    np.testing.assert_allclose(st[th0:th0 + L], rst[th0:th0 + L], rtol=REL_TOL, atol=0)
    assert not len(mismatch(tw, rtw)), f"{what}: widths differ"
    assert not len(mismatch(ta, rta)), f"{what}: width accumulators differ"


def _sweeps_vs_reference(G, N, seed):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    counts, X, h = heterosis(G, N=N, seed=seed)
    L = X.shape[1]
    cfg = _abi.make_config(chains=2, burnin=200, iterations=100, thin=20, seed=7)
    ref = oracle.RefEngine(counts, X, h, cfg, workers=_threads())
    gpu = Product(counts, X, h, cfg)
    _, T, _ = sizes(G, N, L)
    st = ref.initial_state(1)
    r = (st, np.ones(T), np.zeros(T))
    g = tuple(x.copy() for x in r)
    # burn-in, tuning active (m <= tune_cutoff = 20), then the monitored
    # phase after burn-in: widths frozen
    for m in (1, 2, 201, 202):
        c_ref = ref.iterate(*r, 1, m)
        c_gpu = gpu.iterate(*g, 1, m)
        assert c_ref == c_gpu, f"clamp events at m={m}: {c_gpu} vs {c_ref}"
        _compare(g, r, G, N, L, f"G={G} N={N} m={m}")


def test_config4_g1m_sweeps_match_reference():
    _sweeps_vs_reference(1_000_000, 16, seed=1)


def test_config5_g200k_n64_sweeps_match_reference():
    _sweeps_vs_reference(200_000, 64, seed=1)


def _loopback_ranks(counts, X, h, cfg, world, contrasts=()):
    group = LoopbackGroup(world)
    engines = []
    for r in range(world):
        e = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg, contrasts=list(contrasts))
        e.shard_loopback(r, group)
        engines.append(e)
    outs, errs = [None] * world, [None] * world

    def work(r):
        try:
            outs[r] = engines[r].run()
        except Exception as ex:  # checked by the caller
            errs[r] = ex

    ts = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=900)
    assert not any(t.is_alive() for t in ts), "loopback ranks did not finish"
    return engines, outs, errs


def test_world8_g1m_sharded_run_equals_single_engine():
    """BASELINE configs[3]'s partition: 977 leaves over 8 ranks (123 leaves
    each, the last rank 116), each rank's genes, the replicated
    hyperparameters, accumulators and the heterosis contrast bit-identical
    to one unsharded engine."""
    counts, X, h = heterosis(1_000_000, seed=1)
    L = X.shape[1]
    cfg = RunConfig(chains=2, burnin=12, iterations=10, thin=5, seed=3, save_genes=20)
    cons = [heterosis_contrast()]
    single = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg, contrasts=cons).run()
    engines, outs, errs = _loopback_ranks(counts, X, h, cfg, 8, contrasts=cons)
    assert not any(errs), errs
    assert engines[-1].shard_range[1] == 1_000_000
    for r, (e, out) in enumerate(zip(engines, outs)):
        lo, hi = e.shard_range
        for c in range(2):
            a, b = single[c], out[c]
            for name in ("eps", "gamma", "beta"):
                assert np.array_equal(getattr(a.final_state, name)[lo:hi],
                                      getattr(b.final_state, name)[lo:hi]), (r, c, name)
            for name in ("theta", "sigma"):
                assert np.array_equal(getattr(a.final_state, name),
                                      getattr(b.final_state, name)), (r, c, name)
            assert (a.final_state.nu, a.final_state.tau) == (b.final_state.nu, b.final_state.tau)
            for acc in ("beta_acc", "gamma_acc", "eps_acc"):
                assert np.array_equal(getattr(a, acc).mean[lo:hi], getattr(b, acc).mean[lo:hi])
                assert np.array_equal(getattr(a, acc).meansq[lo:hi],
                                      getattr(b, acc).meansq[lo:hi])
            for acc in ("nu_acc", "tau_acc", "theta_acc", "sigma_acc"):
                assert np.array_equal(getattr(a, acc).mean, getattr(b, acc).mean)
            assert np.array_equal(a.contrasts[0].prob[lo:hi], b.contrasts[0].prob[lo:hi])
    for c in range(2):
        assert sum(o[c].clamp_events for o in outs) == single[c].clamp_events


@pytest.mark.parametrize("max_shrink", [1, 3])
def test_sharded_stall_is_raised_identically_on_every_rank(max_shrink):
    """A stall is recorded on the rank that owns the gene; the gathered
    stall flags stop the chain on every rank, and sync exchanges the records
    so every rank raises the reference's first stall (the one a single
    engine raises: earliest iteration, then the sequential order)."""
    counts, X, h = heterosis(5000, seed=3)
    cfg = RunConfig(chains=2, burnin=30, iterations=30, thin=5, seed=5)
    cfg.slice.max_shrink = max_shrink
    with pytest.raises(SamplerStallError) as one:
        GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg).run()
    _, _, errs = _loopback_ranks(counts, X, h, cfg, 3)
    want = one.value
    for r, ex in enumerate(errs):
        assert isinstance(ex, SamplerStallError), (r, ex)
        assert (ex.step, ex.index1, ex.index2, ex.iteration) == \
            (want.step, want.index1, want.index2, want.iteration), (r, str(ex), str(want))
        assert ex.x0 == want.x0 and ex.width == want.width
        assert str(ex) == str(want)
