"""CPU: assembling a gene-sharded job's results (paper_1606_06659_b200.shards).

Each rank's outputs are a full-size ChainOutput with only its gene range
filled (the layout cmc_engine_get_output gives a shard) and identical
hyperparameters.  merge_shard_outputs must rebuild the unsharded outputs
exactly, and gather_shard_outputs must do so across 2 gloo ranks.  The GPU
side (real shards -> load_outputs -> write_results equal to one unsharded
engine) is tests/test_gpu_loopback.py."""
import copy
import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1606_06659_b200.engine import (ChainOutput, ChainState, ConfigError, ContrastResult,
                                          ContrastSpec, ContrastTerm, Moments, ParamRef)
from paper_1606_06659_b200.shards import gather_shard_outputs, merge_shard_outputs

G, N, L, C = 2600, 4, 3, 2
RANGES2 = [(0, 2048), (2048, 2600)]
RANGES3 = [(0, 1024), (1024, 2048), (2048, 2600)]


def _moments(rng, *shape):
    return Moments(7, *[rng.standard_normal(shape) for _ in range(4)])


def _truth(seed=3):
    rng = np.random.default_rng(seed)
    specs = [ContrastSpec("g", [ContrastTerm([(ParamRef("beta_col", 1), 1.0)], 0.0)], True),
             ContrastSpec("h", [ContrastTerm([(ParamRef("theta", 1), 1.0)], 0.0)], False)]
    saved = np.array([5, 1500, 2100, 2599])
    ncols = 2 + 2 * L + len(saved) * (L + 1)
    outs = []
    for c in range(C):
        st = ChainState(G, N, L, xi=True)
        st.eps, st.gamma = rng.standard_normal((G, N)), rng.random(G) + 0.5
        st.beta, st.xi = rng.standard_normal((G, L)), rng.random((G, L)) + 0.1
        st.theta, st.sigma, st.nu, st.tau = rng.standard_normal(L), rng.random(L), 3.0, 0.5
        outs.append(ChainOutput(
            c, _moments(rng, 1), _moments(rng, 1), _moments(rng, L), _moments(rng, L),
            _moments(rng, G, L), _moments(rng, G), _moments(rng, G, N),
            [ContrastResult(specs[0], 7, rng.random(G)), ContrastResult(specs[1], 7, rng.random(1))],
            [f"c{k}" for k in range(ncols)], rng.standard_normal((ncols, 3)),
            np.array([10, 20, 30]), saved.copy(), np.zeros(7), 40 + c, st, _moments(rng, G, L)))
    return outs


def _shard_view(truth, lo, hi, clamps):
    """What rank [lo, hi) returns: gene rows outside the range are zero."""
    outs = []
    for o in truth:
        s = copy.deepcopy(o)
        out_of = np.ones(G, bool)
        out_of[lo:hi] = False
        for name in ("beta_acc", "gamma_acc", "eps_acc", "xi_acc"):
            for k in ("mean", "meansq", "mean_c", "meansq_c"):
                getattr(getattr(s, name), k)[out_of] = 0.0
        for name in ("eps", "gamma", "beta", "xi"):
            getattr(s.final_state, name)[out_of] = 0.0
        s.contrasts[0].prob[out_of] = 0.0
        for k, g in enumerate(s.saved_genes):
            if not lo <= g < hi:
                c0 = 2 + 2 * L + k * (L + 1)
                s.samples[c0:c0 + L + 1] = 0.0
        s.clamp_events = clamps
        outs.append(s)
    return outs


def _assert_equal(a, b):
    for name in ("nu_acc", "tau_acc", "theta_acc", "sigma_acc", "beta_acc", "gamma_acc",
                 "eps_acc", "xi_acc"):
        for k in ("mean", "meansq", "mean_c", "meansq_c"):
            assert np.array_equal(getattr(getattr(a, name), k), getattr(getattr(b, name), k)), name
    for name in ("eps", "gamma", "beta", "xi", "theta", "sigma"):
        assert np.array_equal(getattr(a.final_state, name), getattr(b.final_state, name)), name
    assert (a.final_state.nu, a.final_state.tau) == (b.final_state.nu, b.final_state.tau)
    for x, y in zip(a.contrasts, b.contrasts):
        assert np.array_equal(x.prob, y.prob)
    assert np.array_equal(a.samples, b.samples)
    assert a.clamp_events == b.clamp_events


@pytest.mark.parametrize("ranges", [RANGES2, RANGES3])
def test_merge_rebuilds_unsharded_outputs(ranges):
    truth = _truth()
    split = [10, 25, 5][:len(ranges)]
    for o in truth:
        o.clamp_events = sum(split)
    per_rank = [_shard_view(truth, lo, hi, split[r]) for r, (lo, hi) in enumerate(ranges)]
    merged = merge_shard_outputs(per_rank, ranges)
    for a, b in zip(merged, truth):
        _assert_equal(a, b)


def test_merge_refuses_ranks_of_different_jobs():
    a, b = _truth(3), _truth(4)
    with pytest.raises(ConfigError):
        merge_shard_outputs([_shard_view(a, 0, 2048, 1), _shard_view(b, 2048, G, 1)], RANGES2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    truth = _truth()
    for o in truth:
        o.clamp_events = 12
    lo, hi = RANGES2[rank]
    mine = _shard_view(truth, lo, hi, 6)
    eng = SimpleNamespace(shard_range=(lo, hi), G=G)
    merged = gather_shard_outputs(eng, mine)
    if rank == 0:
        for a, b in zip(merged, truth):
            _assert_equal(a, b)
        result[0] = "ok"
    else:
        result[1] = "none" if merged is None else "unexpected"
    dist.destroy_process_group()


def test_gather_over_two_gloo_ranks():
    port = _free_port()
    with mp.Manager() as m:
        result = m.dict()
        mp.spawn(_worker, args=(2, port, result), nprocs=2, join=True)
        assert dict(result) == {0: "ok", 1: "none"}
