"""Development aid: device ms per 4-chain sweep, unsharded engine vs the same
engine as a 1-rank NCCL clique (split tail: separate hyper kernels after the
all-gathers), at the Paschold shape and at G = 1M."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from ctypes import byref
from paper_1606_06659_b200 import (builtin_design, generate, SimSpec, GibbsEngine, ModelSpec,
                                   RunConfig, CountMatrix, heterosis_contrast)
from paper_1606_06659_b200._abi import CmcError

for G in (39656, 1_000_000):
    X = builtin_design("heterosis16x5", 16)
    counts = generate(SimSpec(G=G, N=16, X=X, nu=8, tau=0.7, theta=[2.5, .2, .2, 0, .1],
                              sigma=[.4, .25, .25, .15, .2], seed=1)).counts
    for sharded in (False, True, False, True):
        eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(16)),
                          RunConfig(chains=4, burnin=100, iterations=200, thin=20, seed=7),
                          contrasts=[heterosis_contrast()])
        if sharded:
            eng.shard(0, 1, GibbsEngine.nccl_unique_id())
        lib, h, err = eng._lib, eng.handle, CmcError()
        assert lib.cmc_engine_begin(h, byref(err)) == 0
        assert lib.cmc_engine_sweeps(h, 1, 151, byref(err)) == 0
        assert lib.cmc_engine_prepare(h, 50, byref(err)) == 0
        assert lib.cmc_engine_sync(h, byref(err)) == 0, err.msg
        s = torch.cuda.ExternalStream(lib.cmc_engine_stream(h))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        assert lib.cmc_engine_sweeps(h, 151, 251, byref(err)) == 0
        e1.record(s)
        assert lib.cmc_engine_sync(h, byref(err)) == 0, err.msg
        torch.cuda.synchronize()
        print(f"G={G} sharded={sharded}: {e0.elapsed_time(e1) / 100:.4f} ms/sweep", flush=True)
        del eng
