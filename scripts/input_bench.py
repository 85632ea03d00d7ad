"""Input-side timing: counts CSV load + median-of-ratios offsets at G genes,
product host loader (cmc_counts_load / cmc_estimate_offsets) against the
reference's load_counts / estimate_offsets (oracle/_ref, single thread as
the reference runs them).  Prints one JSON line.

  python scripts/input_bench.py [--genes 1000000] [--samples 16]
"""
import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402  (checker + reference arm only)
from paper_1606_06659_b200 import estimate_offsets, load_counts  # noqa: E402


def best(fn, reps):
    t = []
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        t.append(time.perf_counter() - t0)
    return min(t), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--genes", type=int, default=1_000_000)
    ap.add_argument("--samples", type=int, default=16)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    rng = np.random.default_rng(1)
    counts = rng.poisson(rng.gamma(2.0, 100.0, size=(a.genes, 1)),
                         size=(a.genes, a.samples)).astype(np.int64)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "counts.csv")
        with open(path, "w") as f:
            f.write("gene," + ",".join(f"s{n + 1}" for n in range(a.samples)) + "\n")
            np.savetxt(f, counts, fmt="%d", delimiter=",",
                       header="", comments="")
        # prefix gene labels: rewrite with labels (savetxt has no row names)
        with open(path) as f:
            lines = f.read().splitlines()
        with open(path, "w") as f:
            f.write(lines[0] + "\n")
            f.write("\n".join(f"g{i + 1},{ln}" for i, ln in enumerate(lines[1:])) + "\n")
        size = os.path.getsize(path)
        t_ours, m = best(lambda: load_counts(path), a.reps)
        t_ref, r = best(lambda: oracle.ref_load_counts(path), a.reps)
        assert np.array_equal(m.counts, r[0]) and m.genes == r[1]
    t_off, h = best(lambda: estimate_offsets(counts), a.reps)
    t_roff, rh = best(lambda: oracle.ref_estimate_offsets(counts), a.reps)
    assert np.array_equal(h.view(np.int64), rh.view(np.int64))
    print(json.dumps({
        "genes": a.genes, "samples": a.samples, "csv_bytes": size,
        "threads": os.cpu_count(),
        "load_s": round(t_ours, 4), "load_ref_s": round(t_ref, 4),
        "load_speedup": round(t_ref / t_ours, 2),
        "load_GBps": round(size / t_ours / 1e9, 3),
        "offsets_s": round(t_off, 4), "offsets_ref_s": round(t_roff, 4),
        "offsets_speedup": round(t_roff / t_off, 2),
        "parity": "counts/labels equal, offsets bit-identical",
    }))


if __name__ == "__main__":
    main()
