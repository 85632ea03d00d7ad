"""Output-side timing: write_results at G genes, 4 chains.  Ours = device
diagnostics + D2H + parallel host formatting (GibbsEngine.write_results);
reference = its own write_results on its own ChainOutputs (oracle/_ref),
timed inside the shim (excludes its run()).  Checks gene_estimates.csv is
byte-identical.  Prints one JSON line.

  python scripts/output_bench.py [--genes 39656] [--iterations 40]
"""
import argparse
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402  (checker + reference arm only)
from paper_1606_06659_b200 import (CountMatrix, GibbsEngine, ModelSpec, RunConfig,  # noqa: E402
                                   SimSpec, builtin_design, generate, heterosis_contrast)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--genes", type=int, default=39656)
    ap.add_argument("--burnin", type=int, default=20)
    ap.add_argument("--iterations", type=int, default=40)
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    X = builtin_design("heterosis16x5", 16)
    counts = generate(SimSpec(G=a.genes, N=16, X=X, nu=8.0, tau=0.7,
                              theta=[2.5, 0.2, 0.2, 0.0, 0.1],
                              sigma=[0.4, 0.25, 0.25, 0.15, 0.2], seed=1)).counts
    cfg = RunConfig(chains=4, burnin=a.burnin, iterations=a.iterations, thin=10, seed=7,
                    save_genes=20)
    het = heterosis_contrast()
    het.id = "c1"
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, [0.0] * 16), cfg, contrasts=[het])
    eng.run()
    out = {"genes": a.genes, "chains": 4, "threads": os.cpu_count()}
    with tempfile.TemporaryDirectory() as d:
        eng.write_results(os.path.join(d, "warm"))
        t0 = time.perf_counter()
        eng.write_results(os.path.join(d, "ours"), wall_seconds=1.0)
        out["write_s"] = round(time.perf_counter() - t0, 4)
        sizes = sum(os.path.getsize(os.path.join(r, f))
                    for r, _, fs in os.walk(os.path.join(d, "ours")) for f in fs)
        out["bytes"] = sizes
        if not a.no_ref:
            ref = oracle.RefEngine(counts, X, [0.0] * 16, cfg.to_c(), contrasts=[het.flat()])
            out["write_ref_s"] = round(ref.write_results(os.path.join(d, "ref"),
                                                         wall_seconds=1.0), 4)
            out["speedup"] = round(out["write_ref_s"] / out["write_s"], 2)
            same = open(os.path.join(d, "ours", "gene_estimates.csv"), "rb").read() == \
                open(os.path.join(d, "ref", "gene_estimates.csv"), "rb").read()
            out["gene_estimates_identical"] = same
    print(json.dumps(out))


if __name__ == "__main__":
    main()
