"""Development aid: device-timed sweep-kernel vs tail time (cmc_engine_profile)
at the bench shape, for A/B of library builds (CMC_LIB_OVERRIDE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ctypes import byref, c_double
from paper_1606_06659_b200 import *
from paper_1606_06659_b200._abi import CmcError
X = builtin_design("heterosis16x5", 16)
counts = generate(SimSpec(G=39656, N=16, X=X, nu=8, tau=0.7, theta=[2.5,.2,.2,0,.1], sigma=[.4,.25,.25,.15,.2], seed=1)).counts
eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(16)), RunConfig(chains=4, burnin=200, iterations=400, thin=20, seed=7), contrasts=[heterosis_contrast()])
lib, h, err = eng._lib, eng.handle, CmcError()
lib.cmc_engine_begin(h, byref(err)); lib.cmc_engine_sweeps(h, 1, 206, byref(err)); lib.cmc_engine_sync(h, byref(err))
g, t = c_double(), c_double()
assert lib.cmc_engine_profile(h, 206, 20, byref(g), byref(t), byref(err)) == 0, err.msg
print(f"kernels {g.value:.4f} ms tail {t.value:.4f} ms", flush=True)
