"""Development aid: the end-to-end run() split into create / begin /
sweeps / outputs, with the previous engine destroyed outside the clock."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ctypes import byref
from paper_1606_06659_b200 import (builtin_design, generate, SimSpec, GibbsEngine, ModelSpec,
                                   RunConfig, CountMatrix, heterosis_contrast)
from paper_1606_06659_b200._abi import CmcError
G, N = 39656, 16
X = builtin_design("heterosis16x5", N)
counts = generate(SimSpec(G=G, N=N, X=X, nu=8, tau=0.7, theta=[2.5, .2, .2, 0, .1],
                          sigma=[.4, .25, .25, .15, .2], seed=1)).counts
import torch; torch.zeros(1, device="cuda")
B, E = int(os.environ.get("E2E_B", "2000")), int(os.environ.get("E2E_E", "4000"))
for rep in range(4):
    gc.collect()
    t0 = time.perf_counter()
    eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(N)),
                      RunConfig(chains=4, burnin=B, iterations=E, thin=20, seed=7, save_genes=20),
                      contrasts=[heterosis_contrast()])
    t1 = time.perf_counter()
    lib, h, err = eng._lib, eng.handle, CmcError()
    assert lib.cmc_engine_begin(h, byref(err)) == 0
    t2 = time.perf_counter()
    assert lib.cmc_engine_sweeps(h, 1, B + E + 1, byref(err)) == 0
    t3 = time.perf_counter()
    assert lib.cmc_engine_sync(h, byref(err)) == 0
    t4 = time.perf_counter()
    outs = [eng._output(c) for c in range(4)]
    t5 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} begin {1e3*(t2-t1):.1f} sweeps-enqueue {1e3*(t3-t2):.1f} "
          f"sync {1e3*(t4-t3):.1f} outputs {1e3*(t5-t4):.1f} total {1e3*(t5-t0):.1f} ms", flush=True)
    del outs, eng

# output copy: fresh (lazily zeroed) arrays vs pre-faulted arrays
import ctypes
from ctypes import c_uint64
from paper_1606_06659_b200._abi import CmcOutputView, dptr, lptr, sizes
eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(N)),
                  RunConfig(chains=4, burnin=20, iterations=40, thin=20, seed=7, save_genes=20),
                  contrasts=[heterosis_contrast()])
outs = eng.run()
S, _, A = sizes(G, N, 5, False)
def view_for(prefault):
    mk = (lambda n: np.ones(n)) if prefault else (lambda n: np.zeros(n))
    accs = [mk(A) for _ in range(4)]
    final = mk(S)
    keep = [accs, final, np.zeros(1, np.int64), np.zeros(G + 10), np.zeros(4, np.int64),
            np.zeros(eng.n_cols * eng.n_rows + 1), np.zeros(eng.n_rows + 1, np.int64),
            np.zeros(1, np.uint64), np.zeros(7)]
    v = CmcOutputView(lptr(keep[2]), dptr(accs[0]), dptr(accs[1]), dptr(accs[2]), dptr(accs[3]),
                      dptr(keep[3]), lptr(keep[4]), dptr(keep[5]), lptr(keep[6]),
                      keep[7].ctypes.data_as(ctypes.POINTER(c_uint64)), dptr(final), dptr(keep[8]))
    return v, keep
err = CmcError()
for pf in (False, True, False, True):
    vs = [view_for(pf) for _ in range(4)]
    t0 = time.perf_counter()
    for c in range(4):
        assert eng._lib.cmc_engine_get_output(eng.handle, c, byref(vs[c][0]), byref(err)) == 0
    t1 = time.perf_counter()
    print(f"get_output x4 prefaulted={pf}: {1e3*(t1-t0):.1f} ms", flush=True)
t0 = time.perf_counter(); o = [eng._output(c) for c in range(4)]; t1 = time.perf_counter()
print(f"_output x4 (python wrapper, fresh arrays): {1e3*(t1-t0):.1f} ms")

# the bench's e2e: GibbsEngine(...).run() from host arrays, engine deleted outside the clock
del eng, o
for rep in range(4):
    gc.collect()
    t0 = time.perf_counter()
    e2 = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(N)),
                     RunConfig(chains=4, burnin=B, iterations=E, thin=20, seed=7, save_genes=20),
                     contrasts=[heterosis_contrast()])
    outs = e2.run()
    t1 = time.perf_counter()
    print(f"run() e2e {1e3*(t1-t0):.1f} ms", flush=True)
    del e2, outs
