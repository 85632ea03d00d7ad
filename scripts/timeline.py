"""Warp-level kernel timeline of a few sweeps (cmc_engine_trace), printed as
per-launch [start, end] intervals per lane: shows the real overlap of the
eps / gene / leaf kernels in the two-lane, two-stream schedule."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from ctypes import byref, c_long
from paper_1606_06659_b200 import (builtin_design, generate, SimSpec, GibbsEngine, ModelSpec,
                                   RunConfig, CountMatrix, heterosis_contrast)
from paper_1606_06659_b200._abi import CmcError

G = int(sys.argv[1]) if len(sys.argv) > 1 else 39656
C = int(sys.argv[2]) if len(sys.argv) > 2 else 4
N = 16
X = builtin_design("heterosis16x5", N)
counts = generate(SimSpec(G=G, N=N, X=X, nu=8, tau=0.7, theta=[2.5,.2,.2,0,.1], sigma=[.4,.25,.25,.15,.2], seed=1)).counts
eng = GibbsEngine(CountMatrix(counts), ModelSpec(X, np.zeros(N)), RunConfig(chains=C, burnin=200, iterations=100, thin=20, seed=7), contrasts=[heterosis_contrast()])
lib, h, err = eng._lib, eng.handle, CmcError()
assert lib.cmc_engine_begin(h, byref(err)) == 0
assert lib.cmc_engine_sweeps(h, 1, 211, byref(err)) == 0
assert lib.cmc_engine_sync(h, byref(err)) == 0
cap = 2_000_000
buf = np.zeros(3 * cap, dtype=np.uint64)
n = c_long()
S = 3
rc = lib.cmc_engine_trace(h, 211, S, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), cap, byref(n), byref(err))
assert rc == 0, err.msg
r = buf[:3 * n.value].reshape(-1, 3)
kid = (r[:, 0] >> 56).astype(int)
slot = ((r[:, 0] >> 48) & 0xff).astype(int)
t0 = r[:, 1].min()
st = (r[:, 1] - t0) / 1e3
en = (r[:, 2] - t0) / 1e3
names = {1: "eps", 2: "gene", 3: "leaf_a", 4: "leaf_b", 5: "hyper_a", 6: "gene_epi"}
lanes = 2 if C >= 2 else 1
lane = slot * lanes // C
rows = []
for k in names:
    for ln in range(lanes):
        m = (kid == k) & (lane == ln)
        if not m.any():
            continue
        order = np.argsort(st[m])
        s_, e_ = st[m][order], en[m][order]
        # split into launches: a new launch starts after the previous one ended
        cur_s, cur_e, cnt = s_[0], e_[0], 1
        for a, b in zip(s_[1:], e_[1:]):
            if a > cur_e + 1.0:
                rows.append((cur_s, cur_e, names[k], ln, cnt))
                cur_s, cur_e, cnt = a, b, 1
            else:
                cur_e = max(cur_e, b)
                cnt += 1
        rows.append((cur_s, cur_e, names[k], ln, cnt))
rows.sort()
print(f"G={G} chains={C} lanes={lanes}: {S} sweeps, span {en.max():.1f} us ({en.max()/S:.1f} us/sweep)")
for s_, e_, nm, ln, cnt in rows:
    print(f"  lane{ln} {nm:7s} {s_:9.1f} -> {e_:9.1f}  ({e_ - s_:7.1f} us, {cnt} warps)")

m6 = kid == 6
if m6.any():
    d = en[m6] - st[m6]
    print(f"gene-kernel leaf epilogues (last block of each leaf, per warp): {m6.sum()} warps, "
          f"duration mean {d.mean():.1f} us, max {d.max():.1f} us")
