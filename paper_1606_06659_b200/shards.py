"""Results of a gene-sharded job (multi-GPU, one process per GPU).

Each rank's run() returns full-size ChainOutputs in which only its own gene
range [lo, hi) is filled.  The hyperparameters (ν, τ, θ, σ, their
accumulators and thinned columns) are complete and identical on every rank,
because every rank runs the same hyper step on the same gathered sums.
This module assembles the job's outputs on one rank:

* merge_shard_outputs: per-rank outputs + ranges -> one list of ChainOutputs,
  equal to what one unsharded engine's run() returns;
* gather_shard_outputs: the torch.distributed collective around it (outputs
  travel to `dst` as pickled numpy arrays, once per run).

The merged outputs go into an unsharded engine of the full problem through
GibbsEngine.load_outputs, whose diagnostics() and write_results() then
produce the reference's files.  The reference has no sharding, so there is
no reference interface here; the per-gene/hyper split follows its
ChainOutput layout (P:include/countmc/engine.hpp:90-108).
"""
from __future__ import annotations

import copy
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .engine import ChainOutput, ConfigError, GibbsEngine

_GENE_MOMENTS = ("beta_acc", "gamma_acc", "eps_acc", "xi_acc")
_MOMENT_KEYS = ("mean", "meansq", "mean_c", "meansq_c")


def merge_shard_outputs(per_rank: Sequence[Sequence[ChainOutput]],
                        ranges: Sequence[Tuple[int, int]]) -> List[ChainOutput]:
    """Assemble per-rank ChainOutputs (rank order, each with its gene range)
    into the job's outputs.  Gene-indexed arrays take rank r's rows
    [lo_r, hi_r); hyper-level values come from rank 0, after a check that
    every rank agrees on them; clamp events are summed (each rank counts its
    own genes' clamps)."""
    if len(per_rank) != len(ranges) or not per_rank:
        raise ConfigError("need one output list and one gene range per rank")
    chains = len(per_rank[0])
    if any(len(o) != chains for o in per_rank):
        raise ConfigError("ranks disagree on the chain count")
    merged = []
    for c in range(chains):
        base = copy.deepcopy(per_rank[0][c])
        for r in range(1, len(per_rank)):
            o = per_rank[r][c]
            for name in ("nu_acc", "tau_acc", "theta_acc", "sigma_acc"):
                a, b = getattr(base, name), getattr(o, name)
                if not (np.array_equal(a.mean, b.mean) and np.array_equal(a.meansq, b.meansq)):
                    raise ConfigError(f"ranks disagree on {name}: not one sharded job")
        nh = 2 + 2 * len(base.theta_acc.mean)
        L = len(base.theta_acc.mean)
        for r, (lo, hi) in enumerate(ranges):
            o = per_rank[r][c]
            for name in _GENE_MOMENTS:
                dst, src = getattr(base, name), getattr(o, name)
                if dst is None:
                    continue
                for k in _MOMENT_KEYS:
                    getattr(dst, k)[lo:hi] = getattr(src, k)[lo:hi]
            for name in ("eps", "gamma", "beta", "xi"):
                d, s = getattr(base.final_state, name), getattr(o.final_state, name)
                if d is not None:
                    d[lo:hi] = s[lo:hi]
            for rd, rs in zip(base.contrasts, o.contrasts):
                if rd.spec.per_gene:
                    rd.prob[lo:hi] = rs.prob[lo:hi]
            for k, g in enumerate(base.saved_genes):
                if lo <= g < hi:
                    c0 = nh + k * (L + 1)
                    base.samples[c0:c0 + L + 1] = o.samples[c0:c0 + L + 1]
        base.clamp_events = int(sum(per_rank[r][c].clamp_events for r in range(len(per_rank))))
        merged.append(base)
    return merged


def gather_shard_outputs(engine: GibbsEngine, outputs: Sequence[ChainOutput],
                         dst: int = 0, group=None) -> Optional[List[ChainOutput]]:
    """Collective over the job's torch.distributed process group: every rank
    passes its engine (for its shard range) and its run() outputs; rank
    `dst` returns the merged outputs, the others None."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = (tuple(engine.shard_range) if hasattr(engine, "shard_range") else (0, engine.G),
            list(outputs))
    got = [None] * world if rank == dst else None
    dist.gather_object(mine, got, dst=dst, group=group)
    if rank != dst:
        return None
    ranges = [g[0] for g in got]
    return merge_shard_outputs([g[1] for g in got], ranges)
