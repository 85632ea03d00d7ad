"""Development aid: device time of each cmc_engine_sweeps call of a run's
first sweeps (burn-in phases), with host wall time beside it."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from ctypes import byref
from paper_1606_06659_b200 import (builtin_design, generate, SimSpec, GibbsEngine, ModelSpec,
                                   RunConfig, CountMatrix, heterosis_contrast)
from paper_1606_06659_b200._abi import CmcError

G = int(sys.argv[1]) if len(sys.argv) > 1 else 39656
C = int(sys.argv[2]) if len(sys.argv) > 2 else 4
X = builtin_design("heterosis16x5", 16)
counts = generate(SimSpec(G=G, N=16, X=X, nu=8, tau=0.7, theta=[2.5, .2, .2, 0, .1],
                          sigma=[.4, .25, .25, .15, .2], seed=1)).counts
eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(16)),
                  RunConfig(chains=C, burnin=200, iterations=400, thin=20, seed=7),
                  contrasts=[heterosis_contrast()])
lib, h, err = eng._lib, eng.handle, CmcError()
assert lib.cmc_engine_begin(h, byref(err)) == 0
s = torch.cuda.ExternalStream(lib.cmc_engine_stream(h))
for a, b in [(1, 6), (6, 56), (56, 106), (106, 151), (151, 201), (201, 206), (206, 226),
             (226, 246), (246, 296), (296, 346)]:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record(s)
    assert lib.cmc_engine_sweeps(h, a, b, byref(err)) == 0
    e1.record(s)
    assert lib.cmc_engine_sync(h, byref(err)) == 0, err.msg
    torch.cuda.synchronize()
    print(f"sweeps {a:4d}..{b - 1:4d}: {e0.elapsed_time(e1) / (b - a):.4f} ms/sweep device, "
          f"{(time.time() - t0) * 1e3:.1f} ms wall", flush=True)
