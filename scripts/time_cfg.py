"""Development aid: device ms per monitored sweep at (G, chains, N), one
K-sweep call after 105 burn-in sweeps.  usage: time_cfg.py G C N [K]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from ctypes import byref
from paper_1606_06659_b200 import (builtin_design, generate, SimSpec, GibbsEngine, ModelSpec,
                                   RunConfig, CountMatrix, heterosis_contrast)
from paper_1606_06659_b200._abi import CmcError
G, C, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
K = int(sys.argv[4]) if len(sys.argv) > 4 else 20
X = builtin_design("heterosis16x5", N)
counts = generate(SimSpec(G=G, N=N, X=X, nu=8, tau=0.7, theta=[2.5, .2, .2, 0, .1],
                          sigma=[.4, .25, .25, .15, .2], seed=1)).counts
eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(N)),
                  RunConfig(chains=C, burnin=100, iterations=K + 20, thin=20, seed=7),
                  contrasts=[heterosis_contrast()])
lib, h, err = eng._lib, eng.handle, CmcError()
assert lib.cmc_engine_begin(h, byref(err)) == 0
assert lib.cmc_engine_sweeps(h, 1, 106, byref(err)) == 0
assert lib.cmc_engine_prepare(h, K, byref(err)) == 0
s = torch.cuda.ExternalStream(lib.cmc_engine_stream(h))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(2):
    torch.cuda.synchronize()
    e0.record(s)
    m0 = 106 + rep * K
    assert lib.cmc_engine_sweeps(h, m0, m0 + K, byref(err)) == 0
    e1.record(s)
    assert lib.cmc_engine_sync(h, byref(err)) == 0
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    print(f"G={G} C={C} N={N} K={K}: {ms:.4f} ms/sweep, {C * G / ms * 1e3:.3e} gene-iter/s", flush=True)
