"""GPU: the gene-sharded exchange path on one GPU.  shard(0, 1, uid) builds
a 1-rank NCCL clique, so the sweep runs exactly as a rank of a multi-GPU
job does: local leaf sums -> ncclAllGather of the partials (captured in the
CUDA graph) -> standalone hyper kernels.  Results must be bit-identical to
the fused single-GPU path and to the oracle."""
import numpy as np
import pytest

import oracle
from paper_1606_06659_b200 import (CountMatrix, GibbsEngine, ModelSpec, RunConfig,
                                   TuningState, heterosis_contrast)
from paper_1606_06659_b200._abi import sizes

from helpers import heterosis, mismatch

pytestmark = pytest.mark.gpu


def engines(counts, X, h, cfg):
    fused = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg,
                        contrasts=[heterosis_contrast()])
    shard = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg,
                        contrasts=[heterosis_contrast()])
    shard.shard(0, 1, GibbsEngine.nccl_unique_id())
    return fused, shard


def test_exchange_path_run_equals_fused_path():
    counts, X, h = heterosis(2500, seed=4)   # 3 leaves, last one partial
    cfg = RunConfig(chains=2, burnin=30, iterations=60, thin=10, seed=5, save_genes=8)
    fused, shard = engines(counts, X, h, cfg)
    a, b = fused.run(), shard.run()
    for c in range(2):
        assert np.array_equal(a[c].final_state.pack(), b[c].final_state.pack())
        for k in ("mean", "meansq"):
            assert np.array_equal(getattr(a[c].beta_acc, k), getattr(b[c].beta_acc, k))
            assert np.array_equal(getattr(a[c].theta_acc, k), getattr(b[c].theta_acc, k))
            assert np.array_equal(getattr(a[c].nu_acc, k), getattr(b[c].nu_acc, k))
        assert np.array_equal(a[c].samples, b[c].samples)
        assert np.array_equal(a[c].contrasts[0].prob, b[c].contrasts[0].prob)
        assert a[c].clamp_events == b[c].clamp_events


def test_exchange_path_iterate_matches_oracle():
    counts, X, h = heterosis(3000, seed=6)
    cfg = RunConfig(chains=1, burnin=20, iterations=20, seed=3)
    _, shard = engines(counts, X, h, cfg)
    orc = oracle.OracleEngine(counts, X, h, cfg.to_c())
    G, N, L = 3000, 16, 5
    S, T, _ = sizes(G, N, L)
    st = orc.initial_state(0)
    tw, ta = np.ones(T), np.zeros(T)
    gs = shard.initial_state(0)
    tu = TuningState(G, N, L)
    th = slice(G * N + G + G * L, G * N + G + G * L + L)
    for m in range(1, 6):
        orc.iterate(st, tw, ta, 0, m)
        shard.iterate(gs, tu, 0, m)
        p = gs.pack()
        keep = np.ones(S, bool)
        keep[th] = False
        assert not len(mismatch(p[keep], st[keep])), m
        np.testing.assert_allclose(p[th], st[th], rtol=1e-12)
        assert np.array_equal(tu.w, tw) and np.array_equal(tu.w_aux, ta)


def test_exchange_path_two_lanes_with_xi_prior():
    """Four chains: the sharded engine runs two chain lanes, each with its
    own split communicator and its own section of the partial buffers; a xi
    prior adds the xi kernel and the 2 + 2L leaf quantities.  Bit-identical
    to the fused path."""
    from paper_1606_06659_b200 import PriorConfig
    counts, X, h = heterosis(2100, seed=8)
    cfg = RunConfig(chains=4, burnin=20, iterations=30, thin=10, seed=9, save_genes=4)
    spec = lambda: ModelSpec(X, h, PriorConfig(beta_prior=["normal", "laplace", "t",  # noqa: E731
                                                           "horseshoe", "normal"], t_df=3.0))
    fused = GibbsEngine(CountMatrix(counts), spec(), cfg, contrasts=[heterosis_contrast()])
    shard = GibbsEngine(CountMatrix(counts), spec(), cfg, contrasts=[heterosis_contrast()])
    shard.shard(0, 1, GibbsEngine.nccl_unique_id())
    a, b = fused.run(), shard.run()
    # per lane: eps, gene, xi, leaf_a, hyper_a, leaf_b, hyper_b
    assert shard._lib.cmc_engine_launches_per_sweep(shard.handle) == 2 * 7
    for c in range(4):
        assert np.array_equal(a[c].final_state.pack(), b[c].final_state.pack()), c
        assert np.array_equal(a[c].xi_acc.mean, b[c].xi_acc.mean)
        assert np.array_equal(a[c].sigma_acc.mean, b[c].sigma_acc.mean)
        assert np.array_equal(a[c].contrasts[0].prob, b[c].contrasts[0].prob)


def test_exchange_path_stall_equals_fused_path():
    """A stall on the NCCL path: the stall flag goes through the gathered
    partials and the records through the sync-time ncclAllGather of stall
    records; the error equals the fused engine's (and so the reference's
    first stall, tests/test_gpu_parity.py)."""
    from paper_1606_06659_b200 import SamplerStallError
    counts, X, h = heterosis(2500, seed=4)
    cfg = RunConfig(chains=2, burnin=30, iterations=30, thin=10, seed=5)
    cfg.slice.max_shrink = 2
    fused, shard = engines(counts, X, h, cfg)
    with pytest.raises(SamplerStallError) as a:
        fused.run()
    with pytest.raises(SamplerStallError) as b:
        shard.run()
    assert str(a.value) == str(b.value)
    assert (a.value.x0, a.value.width) == (b.value.x0, b.value.width)
