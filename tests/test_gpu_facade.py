"""GPU: the C++ facade (include/countmc_b200.hpp) drives the same engine as
the Python mirror: examples/facade_run.cpp's numbers equal the Python API's
on identical inputs, bit for bit."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_1606_06659_b200 import (CountMatrix, GibbsEngine, ModelSpec, RunConfig,
                                   TuningState, builtin_design)

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_facade_matches_python_mirror(tmp_path):
    exe = os.path.join(ROOT, "paper_1606_06659_b200", "lib", "facade_run")
    out = json.loads(subprocess.run([exe, str(tmp_path / "cpp")], check=True, capture_output=True,
                                    text=True).stdout.strip().splitlines()[-1])
    G, N, L = 300, 16, 5
    X = builtin_design("heterosis16x5", N)
    counts = np.array([[(g * 7 + n * 13) % 41 + (g % 5) * 3 for n in range(N)]
                       for g in range(G)], dtype=np.int64)
    cfg = RunConfig(chains=2, burnin=40, iterations=60, thin=10, seed=11, save_genes=6)
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(N)), cfg)
    st, tu = eng.initial_state(1), TuningState(G, N, L)
    eng.iterate(st, tu, 1, 1)
    outs = eng.run()
    assert out["iter_nu"] == st.nu and out["iter_eps0"] == st.eps[0, 0]
    assert out["nu0"] == outs[0].final_state.nu and out["nu1"] == outs[1].final_state.nu
    bsum = 0.0
    for v in outs[0].beta_acc.mean.ravel():
        bsum += float(v)
    assert out["beta_mean_sum"] == bsum and out["count"] == 60
    eng.write_results(str(tmp_path / "py"))
    for f in ("gene_estimates.csv", "hyper_estimates.csv", "diagnostics.csv",
              "samples/chain_1.csv", "samples/chain_2.csv"):
        assert (tmp_path / "cpp" / f).read_bytes() == (tmp_path / "py" / f).read_bytes(), f
