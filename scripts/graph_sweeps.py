"""Profiling driver: the production schedule (50-sweep CUDA graphs, two
chain lanes) at the bench workload, so `ncu --graph-profiling graph` sees
whole graph replays: 4 burn-in graphs (sweeps 1..200), then 2 monitored
50-sweep graphs (sweeps 201..300)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ctypes import byref
from paper_1606_06659_b200 import (builtin_design, generate, SimSpec, GibbsEngine, ModelSpec,
                                   RunConfig, CountMatrix, heterosis_contrast)
from paper_1606_06659_b200._abi import CmcError

G = int(os.environ.get("G", "39656"))
X = builtin_design("heterosis16x5", 16)
counts = generate(SimSpec(G=G, N=16, X=X, nu=8, tau=0.7, theta=[2.5, .2, .2, 0, .1],
                          sigma=[.4, .25, .25, .15, .2], seed=1)).counts
eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(16)),
                  RunConfig(chains=4, burnin=200, iterations=200, thin=20, seed=7, save_genes=20),
                  contrasts=[heterosis_contrast()])
lib, h, err = eng._lib, eng.handle, CmcError()
assert lib.cmc_engine_begin(h, byref(err)) == 0
assert lib.cmc_engine_sweeps(h, 1, 201, byref(err)) == 0
assert lib.cmc_engine_sweeps(h, 201, 301, byref(err)) == 0
assert lib.cmc_engine_sync(h, byref(err)) == 0, err.msg
print("done")
