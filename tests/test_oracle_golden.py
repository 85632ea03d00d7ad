"""The oracle reproduces, bit for bit, the golden sweeps and run() outputs the
UNMODIFIED reference produced (tests/golden/make_golden.py).  CPU only;
needs no reference sources at run time."""
import os

import numpy as np
import pytest

import oracle
from paper_1606_06659_b200 import _abi

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
KEYS = ["chains", "iterations", "burnin", "tune_cutoff", "thin", "seed",
        "max_step_out", "max_shrink", "w_init", "save_genes", "sampler_mode"]


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def cfg_of(z):
    kw = dict(zip(KEYS, z["cfg"].tolist()))
    for k in KEYS:
        if k != "w_init":
            kw[k] = int(kw[k])
    return _abi.make_config(**kw)


def replay_sweeps(engine_cls, name):
    z = load(name)
    eng = engine_cls(z["counts"], z["X"], z["h"], cfg_of(z))
    chain, m0, m1 = int(z["chain"]), int(z["m0"]), int(z["m1"])
    st = eng.initial_state(chain)
    assert np.array_equal(st, z["init"]), "initial_state differs"
    assert np.array_equal(eng.saved_genes(), z["saved"])
    T = z["tw"].shape[1]
    tw, ta = np.full(T, cfg_of(z).w_init), np.zeros(T)
    out = []
    for k, m in enumerate(range(m0, m1)):
        c = eng.iterate(st, tw, ta, chain, m)
        out.append((st.copy(), tw.copy(), ta.copy(), c))
    return z, out


@pytest.mark.parametrize("name", ["sweeps_heterosis_g40.npz", "sweeps_tiny.npz",
                                  "sweeps_twocol_direct.npz"])
def test_oracle_reproduces_reference_sweeps(name):
    z, out = replay_sweeps(oracle.OracleEngine, name)
    for k, (st, tw, ta, c) in enumerate(out):
        assert np.array_equal(st, z["states"][k]), f"sweep {k}"
        assert np.array_equal(tw, z["tw"][k]) and np.array_equal(ta, z["ta"][k])
        assert c == z["clamps"][k]


def test_oracle_reproduces_reference_run():
    z = load("run_heterosis_g24.npz")
    from helpers import HETEROSIS
    eng = oracle.OracleEngine(z["counts"], z["X"], z["h"], cfg_of(z), contrasts=[HETEROSIS])
    assert np.array_equal(eng.saved_genes(), z["saved"])
    for c in range(int(z["cfg"][0])):
        o = eng.run_chain(c)
        for k in ("count", "mean", "meansq", "prob", "samples", "iters", "clamps", "final"):
            assert np.array_equal(o[k], z[f"c{c}_{k}"]), (c, k)
