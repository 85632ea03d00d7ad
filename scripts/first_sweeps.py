"""Development aid: per-phase device ms of the first 5 sweeps from w_init
(burn-in, tuning active) against 5 steady sweeps after burn-in, 4 chains at
the Paschold shape (cmc_engine_profile_phases)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ctypes import byref, c_double
from paper_1606_06659_b200 import (builtin_design, generate, SimSpec, GibbsEngine, ModelSpec,
                                   RunConfig, CountMatrix, heterosis_contrast)
from paper_1606_06659_b200._abi import CmcError, CMC_PHASES, PHASE_NAMES

X = builtin_design("heterosis16x5", 16)
counts = generate(SimSpec(G=39656, N=16, X=X, nu=8, tau=0.7, theta=[2.5, .2, .2, 0, .1],
                          sigma=[.4, .25, .25, .15, .2], seed=1)).counts
eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(16)),
                  RunConfig(chains=4, burnin=200, iterations=100, thin=20, seed=7),
                  contrasts=[heterosis_contrast()])
lib, h, err = eng._lib, eng.handle, CmcError()
assert lib.cmc_engine_begin(h, byref(err)) == 0
ph = (c_double * CMC_PHASES)()
assert lib.cmc_engine_profile_phases(h, 1, 5, ph, byref(err)) == 0, err.msg
print("first 5", {n: round(ph[i], 4) for i, n in enumerate(PHASE_NAMES)}, flush=True)
assert lib.cmc_engine_sweeps(h, 6, 211, byref(err)) == 0
assert lib.cmc_engine_sync(h, byref(err)) == 0, err.msg
assert lib.cmc_engine_profile_phases(h, 211, 5, ph, byref(err)) == 0, err.msg
print("steady ", {n: round(ph[i], 4) for i, n in enumerate(PHASE_NAMES)}, flush=True)
