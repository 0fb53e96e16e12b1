"""Multi-rank host logic on CPU (gloo, world_size 2): community partitioning,
the uneven all-gather used after every stage, and a sharded RK4 trajectory
(oracle arithmetic standing in for the per-rank stage kernel) equal to the
unsharded one.  The GPU path of the same driver is tested bitwise against a
single rank in tests/test_gpu_multi.py (VirtualCluster)."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_16657_b200 import graph as G
from paper_2203_16657_b200 import multi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_rows_whole_communities_and_balance():
    dec = G.planted_partition_decomposition([50, 400, 30, 250, 90, 300], 0.8, 0.02, 3)
    for world in (1, 2, 3, 4):
        rng = multi.partition_rows(dec, world)
        assert rng[0][0] == 0 and rng[-1][1] == dec.n_nodes
        assert all(a[1] == b[0] for a, b in zip(rng[:-1], rng[1:]))
        off = set(dec.offsets.tolist())
        assert all(lo in off for lo, _ in rng)  # cut at community starts
    cost = multi.row_costs(dec)
    r2 = multi.partition_rows(dec, 2)
    c = [cost[lo:hi].sum() for lo, hi in r2]
    assert max(c) / min(c) < 1.6


@pytest.mark.parametrize("world", [2, 3])
def test_shard_layouts_partition_the_correction(world):
    """Per-rank layouts/schedules together encode exactly the directed S."""
    from paper_2203_16657_b200 import plan as PL

    from test_graph_plan import _schedule_to_directed

    rng = np.random.default_rng(world)
    g, part = G.planted_partition_graph([50, 3, 1, 80, 33, 64], 0.8, 0.05, world)
    a = part.assignment.copy()
    a[rng.choice(a.shape[0], 20, replace=False)] = -1
    used = np.unique(a[a >= 0])
    remap = -np.ones(a.max() + 2, dtype=np.int64)
    remap[used] = np.arange(used.size)
    part = G.Partition.from_assignment(np.where(a >= 0, remap[a], -1))
    dec = G.decompose(g, part)
    rs, cs = [], []
    for lo, hi in multi.partition_rows(dec, world):
        lay = PL.build_layout(dec, row_range=(lo, hi))
        sch = PL.build_schedule(lay, sm_count=3)
        r, c = _schedule_to_directed(lay, sch)
        assert np.all((r >= lo) & (r < hi))
        rs.append(r)
        cs.append(c)
    r, c = np.concatenate(rs), np.concatenate(cs)
    rows, cols, _ = dec.directed()
    n = dec.n_nodes
    assert np.array_equal(np.sort(r * n + c), np.sort(rows * n + cols))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import cia
        from oracle import kernels as K

        # 1. uneven all-gather
        ranges = [(0, 3), (3, 10)]
        buf = torch.full((10, 2), -1.0, dtype=torch.float64)
        lo, hi = ranges[rank]
        buf[lo:hi] = torch.arange(lo, hi, dtype=torch.float64)[:, None] * (rank + 1)
        multi.exchange_slices(buf, ranges, rank)
        ok1 = torch.equal(buf[:3, 0], torch.arange(0, 3, dtype=torch.float64)) and \
            torch.equal(buf[3:, 0], torch.arange(3, 10, dtype=torch.float64) * 2)
        # 2. sharded RK4 with the per-stage exchange (oracle stands in for the kernel)
        dec = G.planted_partition_decomposition([40, 70, 25, 60], 0.85, 0.05, 11)
        n = dec.n_nodes
        rng = np.random.default_rng(5)
        omega = rng.standard_normal(n)
        theta0 = rng.uniform(-math.pi, math.pi, n)
        s = dec.correction
        ranges = multi.partition_rows(dec, world)
        lo, hi = ranges[rank]

        def rhs_own(x):
            k = cia.kuramoto_rhs_cia(K, x, omega, dec.offsets, s.iu, s.iv, s.sgn, 3.0, n)
            out = torch.zeros(n, dtype=torch.float64)
            out[lo:hi] = torch.from_numpy(k[lo:hi])
            return out

        x = torch.from_numpy(theta0.copy())
        dt = 0.01
        for _ in range(5):
            xs = x.clone()
            ksum = torch.zeros(n, dtype=torch.float64)
            stage = xs
            for j, (c, w) in enumerate([(dt / 2, 1.0), (dt / 2, 2.0), (dt, 2.0), (None, 1.0)]):
                k = rhs_own(stage.numpy())
                ksum[lo:hi] += w * k[lo:hi]
                if c is not None:
                    stage = xs.clone()
                    stage[lo:hi] = xs[lo:hi] + c * k[lo:hi]
                    multi.exchange_slices(stage, ranges, rank)  # the per-stage collective
            x = xs.clone()
            x[lo:hi] = torch.from_numpy(cia.wrap_phase((xs[lo:hi] + dt / 6 * ksum[lo:hi]).numpy()))
            multi.exchange_slices(x, ranges, rank)

        def rhs(xx):
            return cia.kuramoto_rhs_cia(K, xx, omega, dec.offsets, s.iu, s.iv, s.sgn, 3.0, n)

        ref, _ = cia.rk4_integrate(rhs, theta0, dt, 5)
        err = float(cia.circ_dist(x.numpy(), ref).max())
        q.put((rank, ok1, err))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_exchange_and_sharded_rk4():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok1, err in res:
        assert ok1, f"rank {rank}: uneven all-gather wrong"
        assert err <= 1e-13, f"rank {rank}: sharded trajectory differs by {err}"


def test_partition_by_cost_generated_case():
    from paper_2203_16657_b200 import gen
    from paper_2203_16657_b200.multi import partition_by_cost

    c = gen.config5()
    off = c.offsets()
    cost = c.row_costs()
    for world in (2, 4, 8):
        ranges = partition_by_cost(off, c.n, cost, world)
        assert ranges[0][0] == 0 and ranges[-1][1] == c.n
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        assert all(lo in set(off.tolist()) for lo, _ in ranges)  # community boundaries
        cum = np.concatenate([[0.0], np.cumsum(cost)])
        share = np.array([cum[hi] - cum[lo] for lo, hi in ranges]) / cum[-1]
        assert share.max() < 1.0 / world * 1.05
