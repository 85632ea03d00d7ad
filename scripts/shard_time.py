import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from ctypes import byref
from paper_1606_06659_b200 import *
from paper_1606_06659_b200._abi import CmcError
X = builtin_design("heterosis16x5", 16)
counts = generate(SimSpec(G=39656, N=16, X=X, nu=8, tau=0.7, theta=[2.5,.2,.2,0,.1], sigma=[.4,.25,.25,.15,.2], seed=1)).counts
for sh in (False, True):
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(16)), RunConfig(chains=4, burnin=200, iterations=200, thin=20, seed=7), contrasts=[heterosis_contrast()])
    if sh: eng.shard(0, 1, GibbsEngine.nccl_unique_id())
    lib, h, err = eng._lib, eng.handle, CmcError()
    lib.cmc_engine_begin(h, byref(err)); lib.cmc_engine_sweeps(h, 1, 206, byref(err)); lib.cmc_engine_sync(h, byref(err))
    s = torch.cuda.ExternalStream(lib.cmc_engine_stream(h)); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(s); assert lib.cmc_engine_sweeps(h, 206, 306, byref(err)) == 0, err.msg; e1.record(s); lib.cmc_engine_sync(h, byref(err)); torch.cuda.synchronize()
    print("shard" if sh else "fused", e0.elapsed_time(e1)/100, "ms/sweep, launches/sweep", lib.cmc_engine_launches_per_sweep(h), flush=True)
