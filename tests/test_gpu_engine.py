"""GPU: the CUDA engine against the reference's golden outputs and the
behaviours P:tests/test_engine.cpp pins, through the mirrored public API
(paper_1606_06659_b200.GibbsEngine).  Slice-sampled values are compared bit
for bit; theta (AS241 tail through log) and conjugate-direct draws within
REL_TOL = 1e-12 (north_star single-sweep tolerance)."""
import numpy as np
import pytest

import oracle
from paper_1606_06659_b200 import (CountMatrix, GibbsEngine, ModelSpec, RunConfig,
                                   SamplerStallError, SliceConfig, TuningState, _abi,
                                   heterosis_contrast)
from paper_1606_06659_b200._abi import sizes

from helpers import HETEROSIS, Product, heterosis, mismatch, simulated, tiny
from test_oracle_golden import cfg_of, load, replay_sweeps

pytestmark = pytest.mark.gpu
REL_TOL = 1e-12


def theta_mask(G, N, L, S):
    m = np.zeros(S, bool)
    o = G * N + G + G * L
    m[o:o + L] = True
    return m


@pytest.mark.parametrize("name", ["sweeps_heterosis_g40.npz", "sweeps_tiny.npz",
                                  "sweeps_twocol_direct.npz"])
def test_gpu_reproduces_reference_golden_sweeps(name):
    z, out = replay_sweeps(Product, name)
    G, N = z["counts"].shape
    L = z["X"].shape[1]
    direct = int(z["cfg"][-1]) == 1
    for k, (st, tw, ta, c) in enumerate(out):
        ref = z["states"][k]
        if direct:
            np.testing.assert_allclose(st, ref, rtol=REL_TOL, atol=0)
        else:
            th = theta_mask(G, N, L, len(st))
            assert not len(mismatch(st[~th], ref[~th])), f"sweep {k}"
            np.testing.assert_allclose(st[th], ref[th], rtol=REL_TOL, atol=0)
        assert not len(mismatch(tw, z["tw"][k])) and not len(mismatch(ta, z["ta"][k]))
        assert c == z["clamps"][k]


def test_gpu_reproduces_reference_golden_run():
    z = load("run_heterosis_g24.npz")
    gpu = Product(z["counts"], z["X"], z["h"], cfg_of(z), contrasts=[HETEROSIS])
    outs = gpu.run()
    G, N = z["counts"].shape
    L = z["X"].shape[1]
    S, _, A = sizes(G, N, L)
    th_acc = np.zeros(A, bool)
    th_acc[2:2 + L] = True
    for c, o in enumerate(outs):
        assert o["count"][0] == z[f"c{c}_count"][0]
        assert o["clamps"][0] == z[f"c{c}_clamps"][0]
        np.testing.assert_array_equal(o["iters"], z[f"c{c}_iters"])
        th = theta_mask(G, N, L, S)
        assert not len(mismatch(o["final"][~th], z[f"c{c}_final"][~th]))
        for k in ("mean", "meansq"):
            assert not len(mismatch(o[k][~th_acc], z[f"c{c}_{k}"][~th_acc])), (c, k)
            np.testing.assert_allclose(o[k], z[f"c{c}_{k}"], rtol=REL_TOL)
        np.testing.assert_allclose(o["samples"], z[f"c{c}_samples"], rtol=REL_TOL)
        np.testing.assert_array_equal(o["prob"], z[f"c{c}_prob"])


# ------------------------------------------------ P:tests/test_engine.cpp

def mk(counts, X, h, **cfg):
    base = dict(chains=1, thin=20, seed=17, save_genes=8)
    base.update(cfg)
    if "burnin" in base and "tune_cutoff" not in base:
        b = base["burnin"]
        base["tune_cutoff"] = b // 10 if b >= 10 else 0
    return GibbsEngine(CountMatrix(counts), ModelSpec(X, h), RunConfig(**base))


def test_invariants_hold_over_a_long_tiny_run():
    """P:tests/test_engine.cpp:87-99"""
    counts, X, h = tiny()
    eng = mk(counts, X, h, burnin=100, iterations=900)
    st = eng.initial_state(0)
    tu = TuningState(1, 1, 1)
    from paper_1606_06659_b200 import PriorConfig
    pr = PriorConfig().resolve(1)
    for m in range(1, 301):
        eng.iterate(st, tu, 0, m)
        st.check(pr)


def test_thinning_and_accumulator_bookkeeping():
    """P:tests/test_engine.cpp:147-169"""
    counts, X, h = simulated(12, 4, 3)
    eng = mk(counts, X, h, burnin=40, iterations=100, thin=20, save_genes=5)
    out = eng.run()[0]
    assert list(out.sample_iters) == [60, 80, 100, 120, 140]
    assert out.samples.shape == (2 + 2 * 2 + 5 * 3, 5)
    assert len(out.sample_names) == 2 + 2 * 2 + 5 * 3
    for acc in (out.nu_acc, out.tau_acc, out.theta_acc, out.beta_acc, out.gamma_acc, out.eps_acc):
        assert acc.count == 100
    assert len(out.saved_genes) == 5 and np.all(np.diff(out.saved_genes) > 0)


def test_beta_columns_update_strictly_one_at_a_time():
    """P:tests/test_engine.cpp:171-182"""
    counts, X, h = simulated(10, 4, 4)
    eng = mk(counts, X, h, burnin=10, iterations=10)
    st, tu, trace = eng.initial_state(0), TuningState(10, 4, 2), []
    eng.iterate(st, tu, 0, 1, step5_trace=trace)
    assert trace == [1, -1, 2, -2]


def test_tuning_freezes_once_burnin_ends():
    """P:tests/test_engine.cpp:184-203"""
    counts, X, h = tiny()
    eng = mk(counts, X, h, burnin=10, iterations=40)
    st, tu = eng.initial_state(0), TuningState(1, 1, 1)
    for m in range(1, 11):
        eng.iterate(st, tu, 0, m)
    w_eps, w_nu, w_sig = tu.width("eps")[0], tu.width("nu")[0], tu.width("sigma")[0]
    assert w_eps != 1.0
    for m in range(11, 51):
        eng.iterate(st, tu, 0, m)
    assert (tu.width("eps")[0], tu.width("nu")[0], tu.width("sigma")[0]) == (w_eps, w_nu, w_sig)


@pytest.mark.parametrize("mode", ["slice_faithful", "conjugate_direct"])
def test_both_sampler_modes_stay_in_support(mode):
    """P:tests/test_engine.cpp:205-216"""
    counts, X, h = simulated(20, 4, 6)
    eng = mk(counts, X, h, burnin=30, iterations=50, sampler_mode=mode)
    out = eng.run()[0]
    from paper_1606_06659_b200 import PriorConfig
    out.final_state.check(PriorConfig().resolve(2))
    assert out.tau_acc.mean[0] > 0 and np.all(out.gamma_acc.mean > 0)


def test_streamed_contrast_equals_thinned_recomputation():
    """P:tests/test_engine.cpp:218-261"""
    from helpers import heterosis
    counts, X, h = heterosis(12, seed=8)
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, h),
                      RunConfig(chains=1, burnin=30, iterations=50, thin=1, seed=17,
                                save_genes=12, tune_cutoff=3),
                      contrasts=[heterosis_contrast()])
    out = eng.run()[0]
    L = 5
    for k, g in enumerate(out.saved_genes):
        b0 = 2 + 2 * L + k * (L + 1)
        b2, b3, b4 = out.samples[b0 + 1], out.samples[b0 + 2], out.samples[b0 + 3]
        recomputed = np.mean((2 * b2 + b4 > 0) & (2 * b3 + b4 > 0))
        assert out.contrasts[0].prob[g] == pytest.approx(recomputed, rel=1e-12, abs=1e-15)


def test_stalled_slice_raises_sampler_stall_error():
    """P:tests/test_engine.cpp:288-301"""
    counts, X, h = simulated(8, 4, 11)
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, h),
                      RunConfig(chains=1, burnin=50, iterations=50, seed=17, tune_cutoff=5,
                                slice=SliceConfig(max_shrink=1)))
    with pytest.raises(SamplerStallError) as e:
        eng.run()
    assert e.value.step and e.value.iteration >= 1 and e.value.step in str(e.value)


def test_batched_chains_equal_chains_run_alone_and_runs_are_deterministic():
    """P:tests/test_engine.cpp:101-129: no scheduling choice (here: how many
    chains share the grid) changes any output bit."""
    counts, X, h = heterosis(300, seed=2)
    cfg = dict(burnin=20, iterations=30, thin=5, seed=9, save_genes=6)
    a = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), RunConfig(chains=2, **cfg),
                    contrasts=[heterosis_contrast()]).run()
    b = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), RunConfig(chains=3, **cfg),
                    contrasts=[heterosis_contrast()]).run()
    for c in range(2):
        assert np.array_equal(a[c].final_state.pack(), b[c].final_state.pack())
        assert np.array_equal(a[c].beta_acc.mean, b[c].beta_acc.mean)
        assert np.array_equal(a[c].eps_acc.meansq, b[c].eps_acc.meansq)
        assert np.array_equal(a[c].samples, b[c].samples)
        assert np.array_equal(a[c].contrasts[0].prob, b[c].contrasts[0].prob)


def test_paschold_shape_trajectory_matches_oracle():
    """30 sweeps at G = 39,656 (BASELINE configs[1]) from chain 1's jittered
    start, burn-in tuning active: every non-theta value bit-identical."""
    counts, X, h = heterosis(39656, seed=1)
    cfg = _abi.make_config(chains=2, burnin=200, iterations=100, seed=7)
    orc = oracle.OracleEngine(counts, X, h, cfg)
    gpu = Product(counts, X, h, cfg)
    G, N, L = 39656, 16, 5
    S, T, _ = sizes(G, N, L)
    st = orc.initial_state(1)
    tw, ta = np.ones(T), np.zeros(T)
    g = (st.copy(), tw.copy(), ta.copy())
    th = theta_mask(G, N, L, S)
    for m in range(1, 31):
        assert orc.iterate(st, tw, ta, 1, m) == gpu.iterate(*g, 1, m)
    assert not len(mismatch(g[0][~th], st[~th]))
    np.testing.assert_allclose(g[0][th], st[th], rtol=REL_TOL)
    assert not len(mismatch(g[1], tw)) and not len(mismatch(g[2], ta))


def test_g1m_properties():
    """BASELINE configs[3] size on one GPU: finite, in support, and the same
    bits on a repeated run (determinism at full size)."""
    counts, X, h = heterosis(1_000_000, seed=1)
    cfg = RunConfig(chains=1, burnin=20, iterations=10, thin=5, seed=3, save_genes=20)
    outs = [GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg).run()[0] for _ in range(2)]
    a, b = outs
    from paper_1606_06659_b200 import PriorConfig
    a.final_state.check(PriorConfig().resolve(5))
    assert np.array_equal(a.final_state.pack(), b.final_state.pack())
    assert np.array_equal(a.beta_acc.mean, b.beta_acc.mean)
    assert a.clamp_events == b.clamp_events


def test_iterate_after_run_leaves_the_run_untouched():
    """iterate() works on caller-owned state (the reference's contract): on
    the device it uses a scratch slot and restores the iteration counter, so
    a finished run()'s outputs and diagnostics are unchanged by it."""
    counts, X, h = heterosis(300, seed=2)
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, h),
                      RunConfig(chains=2, burnin=20, iterations=30, thin=10, seed=4))
    outs = eng.run()
    d0 = eng.diagnostics()
    st, tu = eng.initial_state(0), eng.tuning_state()
    for m in range(1, 4):
        eng.iterate(st, tu, 0, m)
    d1 = eng.diagnostics()
    assert np.array_equal(d0.rhat, d1.rhat)
    for c in range(2):
        fresh = eng._output(c)
        assert np.array_equal(fresh.final_state.pack(), outs[c].final_state.pack())
        assert np.array_equal(fresh.beta_acc.mean, outs[c].beta_acc.mean)
    # and the iterate sweeps equal the oracle's from the same start
    orc = oracle.OracleEngine(counts, X, h, RunConfig(chains=2, burnin=20, iterations=30,
                                                      thin=10, seed=4).to_c())
    ost = orc.initial_state(0)
    _, T, _ = sizes(300, 16, 5)
    tw, ta = np.ones(T), np.zeros(T)
    for m in range(1, 4):
        orc.iterate(ost, tw, ta, 0, m)
    th = slice(300 * 16 + 300 + 300 * 5, 300 * 16 + 300 + 300 * 5 + 5)
    p = st.pack()
    keep = np.ones(len(p), bool)
    keep[th] = False
    assert not len(mismatch(p[keep], ost[keep]))


@pytest.mark.parametrize("prior", [None, ["normal", "horseshoe", "t", "laplace", "normal"]])
def test_step_timing_mode_is_bit_identical_and_reports_every_step(prior, tmp_path):
    """The per-step timing mode (reference StepTimings,
    P:src/engine.cpp:173-176): each step launched on its own with events
    between them.  Same results bit for bit; every one of the seven steps
    gets device time (the reference's step order: epsilon, gamma, nu, tau,
    beta, theta, sigma)."""
    from paper_1606_06659_b200 import PriorConfig
    counts, X, h = heterosis(3000, seed=5)
    spec = ModelSpec(X, h, PriorConfig(beta_prior=prior, t_df=3.0)) if prior else ModelSpec(X, h)
    cfg = RunConfig(chains=2, burnin=20, iterations=20, thin=5, seed=9, save_genes=5)
    a = GibbsEngine(CountMatrix(counts), spec, cfg, contrasts=[heterosis_contrast()]).run()
    eng = GibbsEngine(CountMatrix(counts), spec, cfg, contrasts=[heterosis_contrast()])
    eng.set_step_timing(True)
    b = eng.run()
    for c in range(2):
        assert np.array_equal(a[c].final_state.pack(), b[c].final_state.pack())
        assert np.array_equal(a[c].beta_acc.mean, b[c].beta_acc.mean)
        assert np.array_equal(a[c].samples, b[c].samples)
        assert np.array_equal(a[c].contrasts[0].prob, b[c].contrasts[0].prob)
        st = b[c].step_seconds
        assert st.shape == (7,) and np.all(st > 0), st
        # the fused schedule reports one device time under the first step
        assert a[c].step_seconds[0] > 0 and np.all(a[c].step_seconds[1:] == 0)
    # the results writer's run_report.json carries the seven steps
    import json
    eng.write_results(str(tmp_path), wall_seconds=1.0)
    rep = json.loads((tmp_path / "run_report.json").read_text())
    steps = rep["step_seconds"]
    assert set(steps) == {"epsilon", "gamma", "nu", "tau", "beta", "theta", "sigma"}
    assert all(v > 0 for v in steps.values()), steps


def test_sweep_calls_of_any_length_replay_the_same_sweeps():
    """cmc_engine_sweeps replays every sweep from a CUDA graph of the call's
    length (whole 50-sweep graphs plus one of the remainder, LRU cache of 6
    lengths): calls of 1..51 sweeps, more distinct lengths than the cache
    holds, some prepared ahead (cmc_engine_prepare), give the same chains
    bit for bit as one run()."""
    from ctypes import byref
    from paper_1606_06659_b200._abi import CmcError
    counts, X, h = heterosis(2100, seed=3)
    lengths = [1, 2, 3, 5, 7, 11, 13, 50, 51, 3, 1, 7]
    total = sum(lengths)
    cfg = RunConfig(chains=2, burnin=60, iterations=total - 60, thin=4, seed=12, save_genes=6)
    a = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg, contrasts=[heterosis_contrast()])
    ref = a.run()
    b = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg, contrasts=[heterosis_contrast()])
    lib, hd, err = b._lib, b.handle, CmcError()
    assert lib.cmc_engine_begin(hd, byref(err)) == 0
    for n in (13, 51):
        assert lib.cmc_engine_prepare(hd, n, byref(err)) == 0
    m = 1
    for n in lengths:
        assert lib.cmc_engine_sweeps(hd, m, m + n, byref(err)) == 0, err.msg
        m += n
    assert lib.cmc_engine_sync(hd, byref(err)) == 0, err.msg
    for c in range(2):
        o = b._output(c)
        assert np.array_equal(o.final_state.pack(), ref[c].final_state.pack())
        assert np.array_equal(o.beta_acc.mean, ref[c].beta_acc.mean)
        assert np.array_equal(o.eps_acc.meansq, ref[c].eps_acc.meansq)
        assert np.array_equal(o.samples, ref[c].samples)
        assert np.array_equal(o.contrasts[0].prob, ref[c].contrasts[0].prob)


def test_progress_callback_reports_every_chain_and_keeps_results():
    """set_progress (P:include/countmc/engine.hpp:138-139): run() then
    enqueues its sweeps in chunks and reports (chain, m, total) after each;
    the chains are the same bits as a run without a callback."""
    counts, X, h = heterosis(1500, seed=4)
    cfg = RunConfig(chains=3, burnin=400, iterations=700, thin=10, seed=6)
    plain = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg).run()
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg)
    seen = []
    eng.set_progress(lambda c, m, total: seen.append((c, m, total)))
    outs = eng.run()
    total = 1100
    assert {c for c, _, _ in seen} == {0, 1, 2}
    for c in range(3):
        ms = [m for cc, m, t in seen if cc == c]
        assert ms == sorted(ms) and ms[-1] == total
        assert all(t == total for cc, _, t in seen if cc == c)
        assert np.array_equal(outs[c].final_state.pack(), plain[c].final_state.pack())
        assert np.array_equal(outs[c].beta_acc.mean, plain[c].beta_acc.mean)
