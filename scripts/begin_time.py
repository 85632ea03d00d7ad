import sys, time, ctypes
sys.path.insert(0, '.')
import numpy as np
from ctypes import byref
from paper_1606_06659_b200 import *
from paper_1606_06659_b200._abi import CmcError, sizes
X = builtin_design("heterosis16x5", 16)
counts = generate(SimSpec(G=39656, N=16, X=X, nu=8, tau=0.7, theta=[2.5,.2,.2,0,.1], sigma=[.4,.25,.25,.15,.2], seed=1)).counts
import torch; torch.zeros(1, device="cuda")
for rep in range(3):
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(16)), RunConfig(chains=4, burnin=2000, iterations=4000, thin=20, seed=7), contrasts=[heterosis_contrast()])
    lib, h, err = eng._lib, eng.handle, CmcError()
    S, T, A = sizes(39656, 16, 5)
    st = np.zeros(S)
    t0 = time.perf_counter(); [lib.cmc_engine_initial_state(h, c, st.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), byref(err)) for c in range(4)]; t1 = time.perf_counter()
    assert lib.cmc_engine_begin(h, byref(err)) == 0; t2 = time.perf_counter()
    assert lib.cmc_engine_begin(h, byref(err)) == 0; t3 = time.perf_counter()
    print(f"4 host initial states {t1-t0:.3f}s  first begin {t2-t1:.3f}s  second begin {t3-t2:.3f}s", flush=True)
    del eng
