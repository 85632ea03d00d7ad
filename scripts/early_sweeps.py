"""Development aid: device ms per sweep over the phases of a default run (widths fixed at w_init until tune_cutoff = 200, then tuned burn-in, then monitored)."""
import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from ctypes import byref
from paper_1606_06659_b200 import (builtin_design, generate, SimSpec, GibbsEngine, ModelSpec, RunConfig, CountMatrix, heterosis_contrast)
from paper_1606_06659_b200._abi import CmcError
X = builtin_design("heterosis16x5", 16)
counts = generate(SimSpec(G=39656, N=16, X=X, nu=8, tau=0.7, theta=[2.5,.2,.2,0,.1], sigma=[.4,.25,.25,.15,.2], seed=1)).counts
eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(16)), RunConfig(chains=4, burnin=2000, iterations=4000, thin=20, seed=7, save_genes=20), contrasts=[heterosis_contrast()])
lib, h, err = eng._lib, eng.handle, CmcError()
assert lib.cmc_engine_begin(h, byref(err)) == 0
s = torch.cuda.ExternalStream(lib.cmc_engine_stream(h))
for a, b in [(1, 201), (201, 401), (401, 2001), (2001, 2201)]:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); assert lib.cmc_engine_sweeps(h, a, b, byref(err)) == 0; e1.record(s)
    assert lib.cmc_engine_sync(h, byref(err)) == 0; torch.cuda.synchronize()
    print(f"sweeps {a}..{b-1}: {e0.elapsed_time(e1)/(b-a):.4f} ms/sweep")
