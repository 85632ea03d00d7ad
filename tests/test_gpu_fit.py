"""GPU: the whole fit flow of the reference CLI (P:tools/main.cpp run_fit:
load_counts -> load_model_matrix -> estimate_offsets -> GibbsEngine::run ->
write_results) done twice on the same CSV files:

* ours: examples/run_fit.cpp, a C++ program on the façade
  (include/countmc_b200.hpp) -- what a reference user's program becomes;
* the reference: its own loaders, offsets, engine and writer (oracle/_ref).

gene_estimates.csv must be byte-identical; the other files cell for cell,
θ-derived cells within 1e-12."""
import csv
import os
import subprocess

import numpy as np
import pytest

import oracle
from paper_1606_06659_b200 import _abi, builtin_design

from helpers import heterosis

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _write_inputs(tmp_path, G=400):
    counts, X, _ = heterosis(G, seed=17)
    cp, xp = tmp_path / "counts.csv", tmp_path / "model_matrix.csv"
    with open(cp, "w") as f:
        f.write("gene," + ",".join(f"s{n + 1}" for n in range(counts.shape[1])) + "\n")
        for g in range(G):
            f.write(f"gene_{g + 1}," + ",".join(str(v) for v in counts[g]) + "\n")
    with open(xp, "w") as f:
        f.write("intercept,parental_hd,hybrid,hybrid_hd,block\n")
        for row in X:
            f.write(",".join(repr(float(v)) for v in row) + "\n")
    return str(cp), str(xp)


def _rows(path):
    return list(csv.reader(open(path, newline="")))


def _theta(name):
    return "theta[" in name


@pytest.mark.usefixtures("ref")
def test_fit_flow_matches_reference_pipeline(tmp_path):
    cp, xp = _write_inputs(tmp_path)
    out_a, out_b = tmp_path / "ours", tmp_path / "ref"
    chains, burnin, iters, thin, seed = 2, 40, 60, 10, 3
    exe = os.path.join(ROOT, "paper_1606_06659_b200", "lib", "run_fit")
    r = subprocess.run([exe, cp, xp, str(out_a), str(chains), str(burnin), str(iters),
                        str(thin), str(seed)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr

    counts, genes, samples, _ = oracle.ref_load_counts(cp)
    X = oracle.ref_load_table(xp, 0)
    h = oracle.ref_estimate_offsets(counts)
    cfg = _abi.make_config(chains=chains, burnin=burnin, iterations=iters, thin=thin, seed=seed)
    oracle.RefEngine(counts, X, h, cfg).write_results(str(out_b), genes=genes)

    assert (out_a / "gene_estimates.csv").read_bytes() == (out_b / "gene_estimates.csv").read_bytes()
    for f in ("hyper_estimates.csv", "diagnostics.csv", "samples/chain_1.csv",
              "samples/chain_2.csv"):
        ra, rb = _rows(out_a / f), _rows(out_b / f)
        assert len(ra) == len(rb) and ra[0] == rb[0], f
        header = ra[0]
        for x, y in zip(ra[1:], rb[1:]):
            for k, (u, v) in enumerate(zip(x, y)):
                if u == v:
                    continue
                assert _theta(x[0]) or _theta(header[k]), (f, x[0], header[k], u, v)
                assert float(u) == pytest.approx(float(v), rel=1e-12, abs=1e-15)
