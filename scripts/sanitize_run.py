"""compute-sanitizer driver (memcheck / racecheck / synccheck): small problems
through every kernel of the product: run() with 2 chains on two lanes and
CUDA graphs (eps, gene with fused leaf sums, hyper_a, leaf_b), a xi-prior
run with a horseshoe column (xi_park_kernel, leaf_a), the per-step timing
mode (split gene kernel), iterate() on the scratch slot, a 1-rank NCCL
clique (hyper kernels after the all-gather), and the device diagnostics."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1606_06659_b200 import (builtin_design, generate, SimSpec, GibbsEngine, ModelSpec,
                                   RunConfig, CountMatrix, PriorConfig, heterosis_contrast)

X = builtin_design("heterosis16x5", 16)
counts = generate(SimSpec(G=2500, N=16, X=X, nu=8, tau=0.7, theta=[2.5, .2, .2, 0, .1],
                          sigma=[.4, .25, .25, .15, .2], seed=1)).counts
h = np.zeros(16)
cfg = RunConfig(chains=2, burnin=60, iterations=50, thin=10, seed=7, save_genes=5)
a = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg, contrasts=[heterosis_contrast()])
a.run()
a.diagnostics()
st, tu = a.initial_state(1), a.tuning_state()
for m in range(1, 3):
    a.iterate(st, tu, 1, m)
b = GibbsEngine(CountMatrix(counts), ModelSpec(X, h, PriorConfig(beta_prior=["normal", "horseshoe", "t", "laplace", "normal"], t_df=3.0)),
                cfg, contrasts=[heterosis_contrast()])
b.run()
c = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg, contrasts=[heterosis_contrast()])
c.set_step_timing(True)
c.run()
d = GibbsEngine(CountMatrix(counts), ModelSpec(X, h), cfg, contrasts=[heterosis_contrast()])
d.shard(0, 1, GibbsEngine.nccl_unique_id())
d.run()
print("sanitize driver done")
