"""Development aid: first sweep at which the device departs from the
oracle for one fuzz case (tests/test_gpu_fuzz.py _case seed), and where."""
import os, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root); sys.path.insert(0, os.path.join(root, "tests"))
import numpy as np
import oracle
from helpers import Product, packed_start, mismatch
from test_gpu_fuzz import _case

seed = int(sys.argv[1])
counts, X, h, cfg, cons, priors = _case(seed)
G, N = counts.shape
L = X.shape[1]
orc = oracle.OracleEngine(counts, X, h, cfg, contrasts=cons, priors=priors)
gpu = Product(counts, X, h, cfg, contrasts=cons, priors=priors)
M = cfg.burnin + cfg.iterations
names = [("eps", G * N), ("gamma", G), ("beta", G * L)]
for c in range(cfg.chains):
    r = packed_start(orc, c, cfg.w_init)
    g = tuple(x.copy() for x in r)
    for m in range(1, M + 1):
        try:
            orc.iterate(*r, c, m)
        except oracle.StallError as e:
            print("oracle stall", c, m, e); break
        try:
            gpu.iterate(*g, c, m)
        except oracle.StallError as e:
            print("device stall", c, m, e); break
        bad = mismatch(g[0], r[0])
        if len(bad):
            i = int(bad[0]); off = 0; where = None
            for nm, k in names:
                if i < off + k:
                    where = (nm, (i - off) // (N if nm == "eps" else (L if nm == "beta" else 1)),
                             (i - off) % (N if nm == "eps" else (L if nm == "beta" else 1)))
                    break
                off += k
            print(f"chain {c} m={m}: {len(bad)} differ, first {i} {where} gpu={g[0][i]!r} orc={r[0][i]!r}")
            if where and where[0] != "eps":
                gg = where[1]
                print("  gene counts max", counts[gg].max(), "sum", counts[gg].sum())
            break
    else:
        print(f"chain {c}: all {M} sweeps equal")
