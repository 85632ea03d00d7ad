"""Profiling driver: horseshoe-prior sweeps (4 chains, Paschold shape)
after burn-in, for ncu on xi_park_kernel (CMC_XI_TRIPS selects the park
budget)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ctypes import byref
from paper_1606_06659_b200 import (builtin_design, generate, SimSpec, GibbsEngine, ModelSpec,
                                   RunConfig, CountMatrix, PriorConfig, heterosis_contrast)
from paper_1606_06659_b200._abi import CmcError

X = builtin_design("heterosis16x5", 16)
counts = generate(SimSpec(G=39656, N=16, X=X, nu=8, tau=0.7, theta=[2.5, .2, .2, 0, .1],
                          sigma=[.4, .25, .25, .15, .2], seed=1)).counts
eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(16), PriorConfig(beta_prior=["horseshoe"])),
                  RunConfig(chains=4, burnin=200, iterations=100, thin=20, seed=7),
                  contrasts=[heterosis_contrast()])
lib, h, err = eng._lib, eng.handle, CmcError()
assert lib.cmc_engine_begin(h, byref(err)) == 0
assert lib.cmc_engine_sweeps(h, 1, 201, byref(err)) == 0
assert lib.cmc_engine_sweeps(h, 201, 203, byref(err)) == 0
assert lib.cmc_engine_sync(h, byref(err)) == 0, err.msg
print("done")
