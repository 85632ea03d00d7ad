"""Gene-sharded multi-rank protocol on CPU (world_size 2, gloo).

Each rank owns the leaf-aligned gene range cmc_shard_bounds() gives it (the
product's own host function), sums its 1024-gene leaves serially, lays the
partials out as the device does ([rank][chain][quantity][leaves_per_rank],
sweep_kernels.cu leaf_part) and all-gathers them; every rank then evaluates
the reference pairwise tree over the gathered leaves and draws the
replicated hyperparameter.  The result must equal the single-process
det_transform_sum (P:include/countmc/parallel.hpp:67-84) bit for bit on
every rank, for any world size: that is what makes the sharded sweep
bit-exact across 1/2/4/8 GPUs."""
import os
import socket
from ctypes import POINTER, byref, c_double, c_long

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

LEAF = 1024


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def serial_sum(x):
    s = 0.0
    for v in x:
        s += float(v)
    return s


def worker(rank, world, port, G, C, Q, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1606_06659_b200 import _abi
    lib = _abi.load_library()
    orc = oracle.load_oracle()
    rng = np.random.default_rng(123)
    data = rng.standard_normal((C, Q, G)) * np.array([1.0, 1e3, 1e-3])[None, :, None]
    lo, hi = c_long(), c_long()
    lib.cmc_shard_bounds(G, rank, world, byref(lo), byref(hi))
    n_leaves = (G + LEAF - 1) // LEAF
    lpr = (n_leaves + world - 1) // world
    part = torch.zeros(world * C * Q * lpr, dtype=torch.float64)
    for c in range(C):
        for q in range(Q):
            for j, g0 in enumerate(range(lo.value, hi.value, LEAF)):
                leaf = g0 // LEAF
                assert leaf // lpr == rank
                part[((rank * C + c) * Q + q) * lpr + (leaf % lpr)] = \
                    serial_sum(data[c, q, g0:min(G, g0 + LEAF)])
    mine = part[rank * C * Q * lpr:(rank + 1) * C * Q * lpr].clone()
    dist.all_gather_into_tensor(part, mine)
    res = np.zeros((C, Q))
    for c in range(C):
        for q in range(Q):
            leaves = np.array([part[((L // lpr * C + c) * Q + q) * lpr + L % lpr].item()
                               for L in range(n_leaves)])
            res[c, q] = orc.orc_pairwise_sum(leaves.ctypes.data_as(POINTER(c_double)), n_leaves)
    # replicated draw at a global site: theta from the reduced sum
    mean, sd = c_double(), c_double()
    orc.orc_theta_fc_params(res[0, 0], G, 0.7, 10.0, byref(mean), byref(sd))
    z = np.zeros(1)
    orc.orc_stream_u01(7, 0, 5, (6 << 56) | 0, 1, z.ctypes.data_as(POINTER(c_double)))
    theta = mean.value + sd.value * orc.orc_normal_quantile(z[0])
    full = np.array([[orc.orc_det_sum(np.ascontiguousarray(data[c, q]).ctypes.data_as(
        POINTER(c_double)), G) for q in range(Q)] for c in range(C)])
    out[rank] = (res.tobytes(), full.tobytes(), theta)
    dist.destroy_process_group()


@pytest.mark.parametrize("G", [5000, 4096, 1500])
def test_sharded_leaf_exchange_is_bit_exact(G):
    world, C, Q = 2, 2, 3
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(worker, args=(world, free_port(), G, C, Q, out), nprocs=world, join=True)
    r0, f0, t0 = out[0]
    r1, f1, t1 = out[1]
    assert r0 == r1 == f0 == f1, "sharded reduction differs from det_transform_sum"
    assert t0 == t1, "replicated hyper draw differs across ranks"


def lane_worker(rank, world, port, G, C, Q, lanes, out):
    """The two-lane layout of the sharded engine (engine.cu
    enqueue_sweep_on): lane k owns chains [slot0, slot0 + n) and the section
    [rank][n][Q][lpr] at offset world * slot0 * Q * lpr of the partial
    buffer, indexed by the lane-relative chain (sweep_kernels.cu PartView);
    each lane all-gathers its own section on its own communicator."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    groups = [dist.new_group(list(range(world))) for _ in lanes]  # ncclCommSplit per lane
    import oracle
    from paper_1606_06659_b200 import _abi
    lib = _abi.load_library()
    orc = oracle.load_oracle()
    rng = np.random.default_rng(321)
    data = rng.standard_normal((C, Q, G))
    lo, hi = c_long(), c_long()
    lib.cmc_shard_bounds(G, rank, world, byref(lo), byref(hi))
    n_leaves = (G + LEAF - 1) // LEAF
    lpr = (n_leaves + world - 1) // world
    buf = torch.zeros(world * C * Q * lpr, dtype=torch.float64)
    res = np.zeros((C, Q))
    for k, (slot0, n) in enumerate(lanes):
        base = world * slot0 * Q * lpr
        for c in range(n):
            for q in range(Q):
                for g0 in range(lo.value, hi.value, LEAF):
                    leaf = g0 // LEAF
                    buf[base + ((rank * n + c) * Q + q) * lpr + leaf % lpr] = \
                        serial_sum(data[slot0 + c, q, g0:min(G, g0 + LEAF)])
        cnt = n * Q * lpr
        sec = buf[base:base + world * cnt]
        mine = sec[rank * cnt:(rank + 1) * cnt].clone()
        dist.all_gather_into_tensor(sec, mine, group=groups[k])
        buf[base:base + world * cnt] = sec
        for c in range(n):
            for q in range(Q):
                leaves = np.array([buf[base + ((L // lpr * n + c) * Q + q) * lpr + L % lpr].item()
                                   for L in range(n_leaves)])
                res[slot0 + c, q] = orc.orc_pairwise_sum(
                    leaves.ctypes.data_as(POINTER(c_double)), n_leaves)
    full = np.array([[orc.orc_det_sum(np.ascontiguousarray(data[c, q]).ctypes.data_as(
        POINTER(c_double)), G) for q in range(Q)] for c in range(C)])
    out[rank] = (res.tobytes(), full.tobytes())
    dist.destroy_process_group()


@pytest.mark.parametrize("G", [5000, 2100])
def test_two_lane_sections_are_bit_exact(G):
    world, C, Q = 2, 4, 3
    lanes = [(0, 2), (2, 2)]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(lane_worker, args=(world, free_port(), G, C, Q, lanes, out), nprocs=world, join=True)
    r0, f0 = out[0]
    r1, f1 = out[1]
    assert r0 == r1 == f0 == f1, "per-lane sharded reduction differs from det_transform_sum"


def ordered_lanes_worker(rank, world, port, sweeps, out):
    """engine.cu enqueue_sweep_on's collective order on 2 ranks: each chain
    lane runs on its own host thread (its own stream), and every all-gather
    first waits for the collective enqueued before it (ev_coll: lane 0's A
    and B, then lane 1's A and B, then the next sweep), so every rank issues
    the gathers in one order.  Here both lanes share ONE process group (the
    strictest case: a communicator needs the same issue order everywhere);
    rank 1 starts its lanes in reverse order with staggered delays, and every
    gathered section must still hold the right lane's, sweep's and phase's
    data."""
    import threading
    import time
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lanes = 2
    # the chain of events: slot k of the global order completes -> k + 1 may go
    order = [(s, lane, ph) for s in range(sweeps) for lane in range(lanes) for ph in "AB"]
    done = [threading.Event() for _ in order]
    got = {}
    errs = []

    def lane_thread(lane):
        try:
            for k, (s, ln, ph) in enumerate(order):
                if ln != lane:
                    continue
                if k > 0:
                    done[k - 1].wait(timeout=60)   # cudaStreamWaitEvent(t, ev_coll)
                mine = torch.tensor([float(rank), float(lane), float(s), float(ph == "B")],
                                    dtype=torch.float64)
                buf = torch.zeros(world * 4, dtype=torch.float64)
                dist.all_gather_into_tensor(buf, mine)
                got[(s, lane, ph)] = buf.view(world, 4).numpy().copy()
                done[k].set()                        # cudaEventRecord(ev_coll, t)
        except Exception as ex:  # reported below
            errs.append(repr(ex))

    ts = [threading.Thread(target=lane_thread, args=(ln,), daemon=True) for ln in range(lanes)]
    starts = list(range(lanes)) if rank == 0 else list(reversed(range(lanes)))
    for i, ln in enumerate(starts):
        ts[ln].start()
        time.sleep(0.05 * (i + rank))
    for t in ts:
        t.join(timeout=120)
    ok = not errs and all(not t.is_alive() for t in ts) and len(got) == len(order)
    if ok:
        for (s, lane, ph), g in got.items():
            want = np.array([[r, lane, s, float(ph == "B")] for r in range(world)])
            ok &= np.array_equal(g, want)
    out[rank] = (ok, errs)
    dist.destroy_process_group()


def test_collective_order_across_lanes_is_rank_independent():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(ordered_lanes_worker, args=(world, free_port(), 4, out), nprocs=world, join=True)
    for r in range(world):
        ok, errs = out[r]
        assert ok, (r, errs)
