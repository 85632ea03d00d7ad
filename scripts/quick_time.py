"""Ad-hoc timing of the sweep (development aid; bench.py is the contract)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from ctypes import byref
from paper_1606_06659_b200 import _abi, builtin_design, generate, SimSpec, GibbsEngine, ModelSpec, RunConfig, CountMatrix
from paper_1606_06659_b200._abi import CmcError

def timeit(G, chains, N=16, burn=200, K=int(os.environ.get("QT_K", "100"))):
    X = builtin_design("heterosis16x5", N)
    counts = generate(SimSpec(G=G, N=N, X=X, nu=8, tau=0.7, theta=[2.5,.2,.2,0,.1], sigma=[.4,.25,.25,.15,.2], seed=1)).counts
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(N)), RunConfig(chains=chains, burnin=burn, iterations=K+10, thin=20, seed=7))
    lib = eng._lib; h = eng.handle; err = CmcError()
    assert lib.cmc_engine_begin(h, byref(err)) == 0, err.msg
    t = time.time()
    assert lib.cmc_engine_sweeps(h, 1, burn + 1, byref(err)) == 0
    assert lib.cmc_engine_sync(h, byref(err)) == 0, err.msg
    tb = time.time() - t
    s = torch.cuda.ExternalStream(lib.cmc_engine_stream(h))
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    assert lib.cmc_engine_sweeps(h, burn + 1, burn + 6, byref(err)) == 0
    assert lib.cmc_engine_prepare(h, K, byref(err)) == 0
    torch.cuda.synchronize()
    e0.record(s)
    assert lib.cmc_engine_sweeps(h, burn + 6, burn + 6 + K, byref(err)) == 0
    e1.record(s)
    assert lib.cmc_engine_sync(h, byref(err)) == 0, err.msg
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    print(f"G={G} N={N} chains={chains}: burn-in {tb/burn*1e3:.3f} ms/sweep, monitored {ms:.4f} ms/sweep, {chains*G/ms*1e3:.3e} gene-iter/s", flush=True)

import sys as _s
CASES = [(39656, 1, 16), (39656, 4, 16), (1000000, 1, 16), (200000, 1, 64)] if len(_s.argv) < 2 else [(39656, 1, 16), (39656, 4, 16)]
for G, C, N in CASES:
    timeit(G, C, N)
