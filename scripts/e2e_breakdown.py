"""Where the end-to-end run() time goes (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ctypes import byref
from paper_1606_06659_b200 import (builtin_design, generate, SimSpec, GibbsEngine, ModelSpec,
                                   RunConfig, CountMatrix, heterosis_contrast)
from paper_1606_06659_b200._abi import CmcError
G, N = 39656, 16
X = builtin_design("heterosis16x5", N)
counts = generate(SimSpec(G=G, N=N, X=X, nu=8, tau=0.7, theta=[2.5,.2,.2,0,.1], sigma=[.4,.25,.25,.15,.2], seed=1)).counts
import torch; torch.cuda.init(); torch.zeros(1, device="cuda")
for B, E in [(200, 500), (2000, 4000), (2000, 4000), (2000, 4000)]:
    t0 = time.perf_counter()
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(N)), RunConfig(chains=4, burnin=B, iterations=E, thin=20, seed=7), contrasts=[heterosis_contrast()])
    t1 = time.perf_counter()
    lib, h, err = eng._lib, eng.handle, CmcError()
    assert lib.cmc_engine_begin(h, byref(err)) == 0
    t2 = time.perf_counter()
    assert lib.cmc_engine_sweeps(h, 1, B + E + 1, byref(err)) == 0
    assert lib.cmc_engine_sync(h, byref(err)) == 0
    t3 = time.perf_counter()
    outs = [eng._output(c) for c in range(4)]
    t4 = time.perf_counter()
    print(f"B={B} E={E}: create {t1-t0:.3f}s begin(+alloc,init states) {t2-t1:.3f}s sweeps {t3-t2:.3f}s outputs {t4-t3:.3f}s total {t4-t0:.3f}s", flush=True)
