"""GPU: one whole run at the reference's DEFAULT RunConfig (4 chains, 2000
burn-in + 4000 iterations, thin 20; P:include/countmc/engine.hpp:22-29) on
the acceptance-c7 data shape (heterosis16x5, G = 1,000), against the
reference's own run() (oracle/_ref, all host threads).

This is the full-chain statement of the north star ("full chains agree on
posterior means and variances") made at the strongest level: 24,000
chain-sweeps, and every accumulator, contrast probability, thinned sample
and final state is bit-identical, θ-derived values within 1e-10."""
import os

import numpy as np
import pytest

import oracle
from paper_1606_06659_b200 import _abi

from helpers import HETEROSIS, Product, heterosis, mismatch

pytestmark = pytest.mark.gpu


LONG = os.environ.get("CMC_LONG") == "1"


@pytest.mark.usefixtures("ref")
@pytest.mark.parametrize("G", [1000, pytest.param(39656, marks=pytest.mark.skipif(
    not LONG, reason="Paschold-size whole run: about 5 minutes of reference time; CMC_LONG=1"))])
def test_default_run_bit_identical_to_reference(G):
    counts, X, h = heterosis(G, seed=99)
    workers = max(1, min(16, os.cpu_count() or 1))
    cfg = _abi.make_config(chains=4, burnin=2000, iterations=4000, thin=20, seed=3,
                           save_genes=20, workers=workers)
    gpu = Product(counts, X, h, cfg, contrasts=[HETEROSIS]).run()
    ref = oracle.RefEngine(counts, X, h, cfg, contrasts=[HETEROSIS], workers=workers).run()
    N, L = 16, 5
    th0 = G * N + G + G * L
    for c in range(4):
        a, b = gpu[c], ref[c]
        assert a["count"][0] == b["count"][0] == 4000
        bad = [i for i in mismatch(a["final"], b["final"]) if not th0 <= i < th0 + L]
        assert not bad, (c, bad[:5])
        np.testing.assert_allclose(a["final"][th0:th0 + L], b["final"][th0:th0 + L], rtol=1e-10)
        for k in ("mean", "meansq"):
            bad = [i for i in mismatch(a[k], b[k]) if not 2 <= i < 2 + L]
            assert not bad, (c, k, bad[:5])
            np.testing.assert_allclose(a[k][2:2 + L], b[k][2:2 + L], rtol=1e-10)
        assert not len(mismatch(a["prob"], b["prob"])), c
        assert a["clamps"][0] == b["clamps"][0]
        # thinned samples: theta columns (2..2+L) to 1e-10, all else exact
        ncols = 2 + 2 * L + 20 * (L + 1)
        sa = a["samples"][:ncols * 200].reshape(ncols, 200)
        sb = b["samples"][:ncols * 200].reshape(ncols, 200)
        keep = [k for k in range(ncols) if not 2 <= k < 2 + L]
        assert not len(mismatch(sa[keep], sb[keep])), c
        np.testing.assert_allclose(sa[2:2 + L], sb[2:2 + L], rtol=1e-10)
