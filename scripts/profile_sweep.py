"""Profiling driver: G genes (default Paschold shape), tuned by burn-in, then
a few directly-launched sweeps (no graph) so ncu sees individual kernels."""
import sys, os, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ctypes import byref
from paper_1606_06659_b200 import builtin_design, generate, SimSpec, GibbsEngine, ModelSpec, RunConfig, CountMatrix
from paper_1606_06659_b200._abi import CmcError

ap = argparse.ArgumentParser()
ap.add_argument("--G", type=int, default=39656)
ap.add_argument("--N", type=int, default=16)
ap.add_argument("--chains", type=int, default=1)
ap.add_argument("--burn", type=int, default=50)
ap.add_argument("--sweeps", type=int, default=3)
a = ap.parse_args()
X = builtin_design("heterosis16x5", a.N)
counts = generate(SimSpec(G=a.G, N=a.N, X=X, nu=8, tau=0.7, theta=[2.5,.2,.2,0,.1], sigma=[.4,.25,.25,.15,.2], seed=1)).counts
eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(a.N)),
                  RunConfig(chains=a.chains, burnin=a.burn, iterations=100, thin=20, seed=7))
lib, h, err = eng._lib, eng.handle, CmcError()
assert lib.cmc_engine_begin(h, byref(err)) == 0, err.msg
assert lib.cmc_engine_sweeps(h, 1, a.burn + 1, byref(err)) == 0
assert lib.cmc_engine_sync(h, byref(err)) == 0, err.msg
for k in range(a.sweeps):   # < 25 per call: direct launches
    assert lib.cmc_engine_sweeps(h, a.burn + 1 + k, a.burn + 2 + k, byref(err)) == 0
assert lib.cmc_engine_sync(h, byref(err)) == 0, err.msg
print("done")
