"""Multi-GPU CIA: community-partitioned row sharding.

* Rows (permuted order) are split into one contiguous range per rank at
  community boundaries, balanced on the planner's cost model; the NONE pool
  may be cut anywhere (32-row granularity).  Communities are never split, so
  every community observable R_c and every intra-community correction is
  rank-local.
* Each rank keeps the full global index space: its DeviceGraph holds only its
  rows (other rows empty), columns stay global, so inter-community neighbours
  are gathered from the rank's full copy of the stage state z.
* After every stage kernel each rank has written z for its own rows; the ranks
  exchange those slices with one group of NCCL broadcasts (an uneven
  all-gather, `exchange_slices`).  That is the only collective: 16 B per node
  per stage.
* Row-owned, fixed-order accumulation + canonical community reductions make
  the trajectory bitwise identical for any rank count (tested with the
  single-GPU `VirtualCluster`, which runs every rank's kernels on one device
  and exchanges by device copies).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .engine import KuramotoEngine
from .errors import BlowUpError, InputError
from .graph import Decomposition
from .plan import INTER_COST, ROW_COST, DeviceGraph

POOL_GRAIN = 32


def row_costs(dec: Decomposition) -> np.ndarray:
    """Per-row cost of the planner's model (padded intra + inter + row overhead)."""
    n = dec.n_nodes
    rows, cols, sg = dec.directed()
    intra = np.bincount(rows[sg < 0], minlength=n)
    inter = np.bincount(rows[sg > 0], minlength=n)
    return (intra + 7) // 8 * 8 + INTER_COST * inter + ROW_COST


def partition_rows(dec: Decomposition, world: int) -> list[tuple[int, int]]:
    """Contiguous row ranges, one per rank, cut at community starts (or in the
    NONE pool at 32-row granularity), balanced on cumulative cost."""
    if world < 1:
        raise InputError("world must be >= 1")
    n = dec.n_nodes
    off = dec.offsets
    cand = list(off[:-1].tolist()) + list(range(int(off[-1]), n, POOL_GRAIN)) + [n]
    cand = np.unique(np.asarray(cand, dtype=np.int64))
    cum = np.concatenate([[0.0], np.cumsum(row_costs(dec))])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        i = int(np.argmin(np.abs(cum[cand] - target)))
        cuts.append(max(int(cand[i]), cuts[-1]))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def exchange_slices(buf, ranges, rank: int, group=None) -> None:
    """Uneven all-gather along dim 0 of ``buf``: rank r owns buf[lo_r:hi_r];
    afterwards every rank holds every slice.  One group of broadcasts."""
    import torch.distributed as dist

    work = []
    for src, (lo, hi) in enumerate(ranges):
        if hi > lo:
            work.append(dist.broadcast(buf[lo:hi], src=src, group=group, async_op=True))
    for w in work:
        w.wait()


def workspace_views(engine: KuramotoEngine):
    """torch views [z0, z1] (float64 [n, 2]) of an engine's workspace."""
    offs = (ctypes.c_int64 * 6)()
    _lib.check(engine.lib.cdk_kuramoto_workspace_layout(ctypes.byref(engine.graph.struct), offs),
               "workspace_layout")
    n = engine.n
    ws = engine.workspace
    views = []
    for k in (0, 1):
        o = int(offs[k])
        views.append(ws[o: o + 16 * n].view(dtype=__import__("torch").float64).view(n, 2))
    return views


class ShardedKuramotoEngine:
    """One rank of a community-sharded Kuramoto CIA trajectory (NCCL exchange)."""

    def __init__(self, dec: Decomposition, omega, coupling: float, norm: float | None, rank: int,
                 world: int, group=None, device=None, ranges=None):
        self.rank, self.world, self.group = rank, world, group
        self.ranges = ranges if ranges is not None else partition_rows(dec, world)
        lo, hi = self.ranges[rank]
        self.graph = DeviceGraph(dec, device=device, row_range=(lo, hi))
        self.eng = KuramotoEngine(dec, omega, coupling=coupling, norm=norm, graph=self.graph)
        self.z = workspace_views(self.eng)

    def _exchange(self, k: int, stream=None) -> None:
        exchange_slices(self.z[k], self.ranges, self.rank, self.group)

    def set_state(self, theta) -> None:
        self.eng.set_state(theta)
        self._exchange(0)

    def rk4(self, dt: float, n_steps: int, stream=None) -> None:
        for _ in range(int(n_steps)):
            for s in range(1, 5):
                self.eng.rk4_stage(dt, s, stream=stream)
                self._exchange(s & 1, stream)
        _lib.check(self.eng.lib.cdk_kuramoto_advance(ctypes.byref(self.graph.struct),
                                                     self.eng.workspace.data_ptr(), int(n_steps),
                                                     _lib.stream_ptr(stream)), "advance")

    def gather_theta(self):
        """Full theta on every rank (own slices exchanged)."""
        th = self.eng.theta.clone()
        exchange_slices(th, self.ranges, self.rank, self.group)
        return th

    def check(self) -> None:
        self.eng.check()


class VirtualCluster:
    """All ranks of a sharded run on ONE device, exchanging by device copies.
    Exercises exactly the per-rank layouts/schedules/kernels of the multi-GPU
    path (for bitwise-equality tests without several GPUs)."""

    def __init__(self, dec: Decomposition, omega, coupling: float, norm: float | None,
                 world: int, device=None):
        self.ranges = partition_rows(dec, world)
        self.ranks = []
        for r in range(world):
            g = DeviceGraph(dec, device=device, row_range=self.ranges[r])
            e = KuramotoEngine(dec, omega, coupling=coupling, norm=norm, graph=g)
            self.ranks.append((e, workspace_views(e)))

    def _exchange(self, k: int) -> None:
        for r, (lo, hi) in enumerate(self.ranges):
            src = self.ranks[r][1][k][lo:hi]
            for q, (_, views) in enumerate(self.ranks):
                if q != r:
                    views[k][lo:hi].copy_(src)

    def set_state(self, theta) -> None:
        for e, _ in self.ranks:
            e.set_state(theta)
        self._exchange(0)

    def rk4(self, dt: float, n_steps: int) -> None:
        for _ in range(int(n_steps)):
            for s in range(1, 5):
                for e, _ in self.ranks:
                    e.rk4_stage(dt, s)
                self._exchange(s & 1)

    def theta(self):
        import torch

        out = torch.empty_like(self.ranks[0][0].theta)
        for (e, _), (lo, hi) in zip(self.ranks, self.ranges):
            out[lo:hi] = e.theta[lo:hi]
        return out

    def check(self) -> None:
        for e, _ in self.ranks:
            st = e.status()
            if st.nonfinite:
                raise BlowUpError(int(st.first_bad_step))


def bench_main(args):
    """bench.py --gpus N under torchrun: config 2 sharded over N ranks."""
    import json
    import os
    import time

    import torch
    import torch.distributed as dist

    from . import configs

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    case = configs.config2()
    dec = case.decomposition()
    omega, theta0 = case.state()
    eng = ShardedKuramotoEngine(dec, omega, case.coupling, case.n, rank, world)
    eng.set_state(theta0)
    W, K = max(3, args.warmup), args.steps
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(W):
        eng.rk4(case.dt, 1)
    eng.set_state(theta0)
    torch.cuda.synchronize()
    dist.barrier()
    cur = torch.cuda.current_stream()
    tot = 0.0
    for _ in range(K):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        eng.rk4(case.dt, 1)
        b.record(cur)
        b.synchronize()
        tot += a.elapsed_time(b)
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([tot], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    eng.check()
    ms = float(t.item())
    if rank == 0:
        print(json.dumps({
            "metric": "node-updates/sec (CIA Kuramoto RK4 RHS)", "value": case.n * K / (ms / 1e3),
            "unit": "node-updates/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2 Kuramoto CIA RK4 sharded by community",
                       "n_nodes": case.n, "parallelism": f"community shards x{world}",
                       "l2": "flushed before every timed step",
                       "ranges": eng.ranges},
            "gpu_launches": 9 * K,
        }), flush=True)
    dist.destroy_process_group()
    time.sleep(0.1)
    return 0
