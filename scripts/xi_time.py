"""Development aid: device ms per sweep of the xi-prior sweeps (first 5
burn-in sweeps from w_init = 1, and steady monitored sweeps), 4 chains at
the Paschold shape."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from ctypes import byref
from paper_1606_06659_b200 import (builtin_design, generate, SimSpec, GibbsEngine, ModelSpec,
                                   RunConfig, CountMatrix, PriorConfig, heterosis_contrast)
from paper_1606_06659_b200._abi import CmcError

X = builtin_design("heterosis16x5", 16)
counts = generate(SimSpec(G=39656, N=16, X=X, nu=8, tau=0.7, theta=[2.5, .2, .2, 0, .1],
                          sigma=[.4, .25, .25, .15, .2], seed=1)).counts
out = {}
for prior in sys.argv[1:] or ["horseshoe", "t", "laplace", "normal"]:
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(16), PriorConfig(beta_prior=[prior], t_df=3.0)),
                      RunConfig(chains=4, burnin=200, iterations=200, thin=20, seed=7),
                      contrasts=[heterosis_contrast()])
    lib, h, err = eng._lib, eng.handle, CmcError()
    assert lib.cmc_engine_begin(h, byref(err)) == 0
    for n in (5, 45, 150, 50):
        assert lib.cmc_engine_prepare(h, n, byref(err)) == 0
    s = torch.cuda.ExternalStream(lib.cmc_engine_stream(h))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(s)
    assert lib.cmc_engine_sweeps(h, 1, 6, byref(err)) == 0
    ev[1].record(s)
    assert lib.cmc_engine_sweeps(h, 6, 251, byref(err)) == 0
    ev[2].record(s)
    assert lib.cmc_engine_sweeps(h, 251, 351, byref(err)) == 0
    ev[3].record(s)
    assert lib.cmc_engine_sync(h, byref(err)) == 0, err.msg
    torch.cuda.synchronize()
    print(f"{prior:10s} first5 {ev[0].elapsed_time(ev[1]) / 5:.4f} ms  steady {ev[2].elapsed_time(ev[3]) / 100:.4f} ms", flush=True)
