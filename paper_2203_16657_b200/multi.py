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
    return partition_by_cost(dec.offsets, dec.n_nodes, row_costs(dec), world)


def partition_by_cost(off, n: int, cost, world: int) -> list[tuple[int, int]]:
    """partition_rows on explicit community offsets and per-row costs (also
    used for device-generated graphs, whose rows never exist on the host)."""
    if world < 1:
        raise InputError("world must be >= 1")
    off = np.asarray(off, dtype=np.int64)
    cand = list(off[:-1].tolist()) + list(range(int(off[-1]), n, POOL_GRAIN)) + [n]
    cand = np.unique(np.asarray(cand, dtype=np.int64))
    cum = np.concatenate([[0.0], np.cumsum(np.asarray(cost, dtype=np.float64))])
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

    def __init__(self, dec: Decomposition | None, omega, coupling: float, norm: float | None,
                 rank: int, world: int, group=None, device=None, ranges=None, graph=None):
        self.rank, self.world, self.group = rank, world, group
        self.ranges = ranges if ranges is not None else partition_rows(dec, world)
        lo, hi = self.ranges[rank]
        self.graph = graph if graph is not None else DeviceGraph(dec, device=device,
                                                                 row_range=(lo, hi))
        self.eng = KuramotoEngine(dec, omega, coupling=coupling, norm=norm, graph=self.graph)
        self.z = workspace_views(self.eng)

    @classmethod
    def generated(cls, case, rank: int, world: int, group=None, device=None):
        """One rank of a device-generated graph (config 5): the rank generates
        only its own rows (gen.generate(row_range=...))."""
        from . import gen

        ranges = partition_by_cost(case.offsets(), case.n, case.row_costs(), world)
        dg, _ = gen.device_graph(case, device, row_range=ranges[rank])
        omega, _ = case.state()
        return cls(None, omega, case.coupling, case.n, rank, world, group, device, ranges, dg)

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

    def __init__(self, dec: Decomposition | None, omega, coupling: float, norm: float | None,
                 world: int, device=None, graphs=None, ranges=None):
        self.ranges = ranges if ranges is not None else partition_rows(dec, world)
        self.ranks = []
        for r in range(world):
            g = (graphs[r] if graphs is not None
                 else DeviceGraph(dec, device=device, row_range=self.ranges[r]))
            e = KuramotoEngine(dec, omega, coupling=coupling, norm=norm, graph=g)
            self.ranks.append((e, workspace_views(e)))

    @classmethod
    def generated(cls, case, world: int, device=None, smem_budget=None):
        """Every rank of a sharded device-generated graph on one device."""
        from . import gen

        ranges = partition_by_cost(case.offsets(), case.n, case.row_costs(), world)
        graphs = [gen.device_graph(case, device, smem_budget=smem_budget, row_range=rr)[0]
                  for rr in ranges]
        omega, _ = case.state()
        return cls(None, omega, case.coupling, case.n, world, device, graphs, ranges)

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
    """bench.py --gpus N under torchrun: config 2 (default) or config 5
    (--config cfg5, each rank generating its own rows) sharded by community
    over N ranks; timed on the device, max over ranks."""
    import json
    import os
    import sys
    import time

    import torch
    import torch.distributed as dist

    from . import configs, gen

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import METRIC, UNIT, ClockSampler, _peaks, algorithmic_bytes_per_rhs  # noqa: E402

    cfg = getattr(args, "config", "cfg2")
    if cfg == "cfg5":
        case = gen.config5()
        omega, theta0 = case.state()
        eng = ShardedKuramotoEngine.generated(case, rank, world)
        nnz_local = eng.graph.layout.nnz_dir
        workload = ("cfg5 Kuramoto CIA RK4, LFR-style N=8000000 (device-generated, each rank its "
                    "own rows), sharded by community")
        flush = None
    else:
        case = configs.config2()
        dec = case.decomposition()
        omega, theta0 = case.state()
        eng = ShardedKuramotoEngine(dec, omega, case.coupling, case.n, rank, world)
        nnz_local = eng.graph.layout.nnz_dir
        workload = "cfg2 Kuramoto CIA RK4, SBM N=200000, sharded by community"
        flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    lib = eng.eng.lib
    nnz_t = torch.tensor([nnz_local], dtype=torch.int64, device="cuda")
    dist.all_reduce(nnz_t)
    nnz = int(nnz_t.item())
    eng.set_state(theta0)
    W, K = max(3, args.warmup), args.steps
    for _ in range(W):
        eng.rk4(case.dt, 1)
    eng.set_state(theta0)
    torch.cuda.synchronize()
    dist.barrier()
    cur = torch.cuda.current_stream()
    tot = 0.0
    sampler = ClockSampler(local)
    l0 = int(lib.cdk_launch_count())
    with sampler:
        for _ in range(K):
            if flush is not None:
                flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(cur)
            eng.rk4(case.dt, 1)
            b.record(cur)
            b.synchronize()
            tot += a.elapsed_time(b)
        torch.cuda.synchronize()
        dist.barrier()
        launches = int(lib.cdk_launch_count()) - l0
        # e2e: host theta0 in, K steps, full theta back on rank 0
        th_h = torch.from_numpy(theta0).pin_memory()
        dist.barrier()
        t0 = time.perf_counter()
        eng.set_state(th_h)
        eng.rk4(case.dt, K)
        final = eng.gather_theta().cpu()
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
    t = torch.tensor([tot, e2e_s * 1e3], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    eng.check()
    ms, e2e_ms = float(t[0].item()), float(t[1].item())
    if rank == 0:
        peak, peak_kind = _peaks()
        b_rhs = algorithmic_bytes_per_rhs(case.n, nnz)
        stage_ms = ms / K / 4.0
        print(json.dumps({
            "metric": METRIC, "value": case.n * K / (ms / 1e3), "unit": UNIT,
            "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms / K,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "n_nodes": case.n, "nnz_dir": nnz,
                       "parallelism": f"community shards x{world} (NCCL all-gather of z per stage)",
                       "l2": "flushed before every timed step" if flush is not None
                       else "inputs >> L2", "ranges": eng.ranges},
            "roofline": {"bound": "hbm", "achieved": b_rhs / world / (stage_ms / 1e3) / 1e9,
                         "peak": peak, "unit": "GB/s", "peak_kind": peak_kind,
                         "frac": b_rhs / world / (stage_ms / 1e3) / 1e9 / peak, "traffic": None,
                         "note": "per GPU: canonical bytes / world over the whole stage "
                                 "(kernels + exchange)"},
            "e2e": {"value": case.n * K / (e2e_ms / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": int(8 * case.n / K),
                    "d2h_bytes_per_step": int(8 * case.n / K)},
            "gpu_launches": launches,
            "clocks": sampler.summary(),
        }), flush=True)
    dist.destroy_process_group()
    time.sleep(0.1)
    return 0
