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
  exchange those slices with one NCCL all-gather of padded equal blocks
  (`exchange_slices`), or — the default when every peer is reachable — the
  stage epilogues store them straight into the peers' buffers over NVLink.  That is the only collective: 16 B per node
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
    afterwards every rank holds every slice.  ONE all-gather of equal,
    padded blocks (max slice length), then one index copy back into place."""
    import torch
    import torch.distributed as dist

    world = len(ranges)
    if world == 1:
        return
    lens = [hi - lo for lo, hi in ranges]
    L = max(max(lens), 1)
    tail = tuple(buf.shape[1:])
    key = (buf.device, buf.dtype, L, tail, tuple(ranges))
    cache = _EXCHANGE_CACHE.get(key)
    if cache is None:
        send = torch.zeros((L,) + tail, dtype=buf.dtype, device=buf.device)
        recv = torch.empty((world * L,) + tail, dtype=buf.dtype, device=buf.device)
        src = torch.cat([torch.arange(r * L, r * L + n) for r, n in enumerate(lens)])
        dst = torch.cat([torch.arange(lo, hi) for lo, hi in ranges])
        cache = (send, recv, src.to(buf.device), dst.to(buf.device))
        _EXCHANGE_CACHE.clear()
        _EXCHANGE_CACHE[key] = cache
    send, recv, src, dst = cache
    lo, hi = ranges[rank]
    send[: hi - lo].copy_(buf[lo:hi])
    dist.all_gather_into_tensor(recv, send, group=group)
    buf.index_copy_(0, dst, recv.index_select(0, src))


_EXCHANGE_CACHE: dict = {}


def workspace_offsets(engine: KuramotoEngine) -> list[int]:
    """byte offsets in an engine's workspace: z0 z1 ksum part0 part1 status peer_bar"""
    offs = (ctypes.c_int64 * 7)()
    _lib.check(engine.lib.cdk_kuramoto_workspace_layout(ctypes.byref(engine.graph.struct), offs),
               "workspace_layout")
    return [int(x) for x in offs]


class PeerTable:
    """Device pointer tables of the fused exchange (include/commdyn_cuda.h
    cdk_peers): every rank's z[0], z[1] and peer-barrier counter.  ``bases``
    are the workspace base addresses of all ranks as seen from this device
    (own workspace, IPC-imported peers, or same-device virtual ranks)."""

    def __init__(self, bases, offsets, rank: int, device, wait: bool):
        """offsets[q]: rank q's workspace_offsets (layouts differ per rank:
        the rblock partial arrays are sized by the rank's own rblocks)."""
        import torch

        n = len(bases)
        z0 = [b + o[0] for b, o in zip(bases, offsets)]
        z1 = [b + o[1] for b, o in zip(bases, offsets)]
        bar = [b + o[6] for b, o in zip(bases, offsets)]
        self._t = [torch.tensor(v, dtype=torch.int64, device=device) for v in (z0, z1, bar)]
        self.struct = _lib.CdkPeers(n_ranks=n, rank=rank, z0=self._t[0].data_ptr(),
                                    z1=self._t[1].data_ptr(), bar=self._t[2].data_ptr(),
                                    bar_base=0, wait=1 if wait else 0)

    def advance(self, n_stages: int) -> None:
        """host-side counter bookkeeping: every stage adds n_ranks to each counter"""
        self.struct.bar_base = (self.struct.bar_base + n_stages * self.struct.n_ranks) & 0xFFFFFFFF


def zero_peer_counter(engine: KuramotoEngine) -> None:
    o = workspace_offsets(engine)[6]
    engine.workspace[o: o + 4].zero_()


def workspace_views(engine: KuramotoEngine):
    """torch views [z0, z1] (float64 [n, 2]) of an engine's workspace."""
    offs = workspace_offsets(engine)
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
                 rank: int, world: int, group=None, device=None, ranges=None, graph=None,
                 p2p: bool = False):
        self.rank, self.world, self.group = rank, world, group
        self.ranges = ranges if ranges is not None else partition_rows(dec, world)
        lo, hi = self.ranges[rank]
        self.graph = graph if graph is not None else DeviceGraph(dec, device=device,
                                                                 row_range=(lo, hi))
        self.eng = KuramotoEngine(dec, omega, coupling=coupling, norm=norm, graph=self.graph)
        self.z = workspace_views(self.eng)
        self.peers = None
        if p2p and world > 1:
            self.peers = self._open_peers_or_fallback()

    def _open_peers_or_fallback(self):
        """all ranks agree: fused exchange if every rank opened its peers,
        otherwise the NCCL all-gather path for everyone"""
        import torch
        import torch.distributed as dist

        try:
            pt, ok = self._open_peers(), 1
        except Exception as exc:  # noqa: BLE001 - any IPC/peer failure -> fallback
            import sys

            print(f"[rank {self.rank}] fused exchange unavailable: {exc}", file=sys.stderr)
            pt, ok = None, 0
        flag = torch.tensor([ok], dtype=torch.int32, device=self.eng.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        return pt if int(flag.item()) == 1 else None

    def _open_peers(self) -> PeerTable:
        """Exchange CUDA IPC handles of every rank's workspace (one
        all_gather_object), open the peers' and build the pointer tables of the
        fused exchange (stage epilogues store into peers over NVLink)."""
        import torch.distributed as dist

        lib = self.eng.lib
        ws = self.eng.workspace.data_ptr()
        h = (ctypes.c_ubyte * 64)()
        off = ctypes.c_uint64()
        _lib.check(lib.cdk_ipc_export(ws, h, ctypes.byref(off)), "ipc_export")
        mine = (bytes(h), int(off.value), workspace_offsets(self.eng))
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=self.group)
        bases, self._imported = [], []
        for q, (hq, oq, _) in enumerate(allh):
            if q == self.rank:
                bases.append(ws)
                continue
            buf = (ctypes.c_ubyte * 64).from_buffer_copy(hq)
            ptr = ctypes.c_void_p()
            _lib.check(lib.cdk_ipc_import(buf, oq, ctypes.byref(ptr)), "ipc_import")
            self._imported.append((ptr.value, oq))
            bases.append(int(ptr.value))
        zero_peer_counter(self.eng)
        import torch

        torch.cuda.synchronize()  # counter zeroed before the agreement all_reduce
        return PeerTable(bases, [a[2] for a in allh], self.rank, self.eng.device, True)

    @classmethod
    def generated(cls, case, rank: int, world: int, group=None, device=None, p2p: bool = False):
        """One rank of a device-generated graph (config 5): the rank generates
        only its own rows (gen.generate(row_range=...))."""
        from . import gen

        ranges = partition_by_cost(case.offsets(), case.n, case.row_costs(), world)
        dg, _ = gen.device_graph(case, device, row_range=ranges[rank])
        omega, _ = case.state()
        return cls(None, omega, case.coupling, case.n, rank, world, group, device, ranges, dg,
                   p2p=p2p)

    def _exchange(self, k: int, stream=None) -> None:
        exchange_slices(self.z[k], self.ranges, self.rank, self.group)

    def set_state(self, theta) -> None:
        self.eng.set_state(theta)
        self._exchange(0)

    def rk4(self, dt: float, n_steps: int, stream=None) -> None:
        if self.peers is not None:  # fused exchange: one persistent launch, NVLink stores
            e = self.eng
            _lib.check(e.lib.cdk_kuramoto_rk4_peers(
                ctypes.byref(self.graph.struct), e.theta.data_ptr(), e.omega.data_ptr(),
                e.k_over_n, float(dt), int(n_steps), e.workspace.data_ptr(),
                ctypes.byref(self.peers.struct), _lib.stream_ptr(stream)), "rk4_peers")
            self.peers.advance(4 * int(n_steps))
            return
        for _ in range(int(n_steps)):
            for s in range(1, 5):
                self.eng.rk4_stage(dt, s, stream=stream)
                self._exchange(s & 1, stream)
            # per step, so a blow-up is reported at its own step (stage
            # kernels count from status.steps_done)
            _lib.check(self.eng.lib.cdk_kuramoto_advance(ctypes.byref(self.graph.struct),
                                                         self.eng.workspace.data_ptr(), 1,
                                                         _lib.stream_ptr(stream)), "advance")

    def verify_fused(self, theta0, dt: float, steps: int = 2) -> str:
        """Run ``steps`` RK4 steps with the fused NVLink exchange and with the
        NCCL all-gather from the same state; keep the fused path only if both
        trajectories are bitwise equal on every rank and no peer-barrier
        watchdog fired (any failure: every rank falls back to NCCL).  Returns
        a one-line verdict for the bench record."""
        import torch
        import torch.distributed as dist

        if self.peers is None:
            return "NCCL all-gather (fused exchange not available)"
        ok, why = 1, ""
        try:
            self.set_state(theta0)
            self.rk4(dt, steps)
            torch.cuda.synchronize()
            if self.eng.status().reserved:
                raise RuntimeError("peer barrier watchdog fired")
            fused = self.gather_theta()
        except Exception as exc:  # noqa: BLE001 - any fused-path failure -> NCCL
            ok, why, fused = 0, str(exc).splitlines()[0][:120], None
        peers, self.peers = self.peers, None
        self.set_state(theta0)
        self.rk4(dt, steps)
        ref = self.gather_theta()
        if ok and not torch.equal(fused, ref):
            ok, why = 0, "fused and NCCL trajectories differ"
        flag = torch.tensor([ok], dtype=torch.int32, device=self.eng.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        if int(flag.item()) == 1:
            self.peers = peers
            return f"fused NVLink exchange (verified bitwise vs NCCL over {steps} steps)"
        return "NCCL all-gather (fused exchange rejected: " + (why or "on another rank") + ")"

    def gather_theta(self):
        """Full theta on every rank (own slices exchanged)."""
        th = self.eng.theta.clone()
        exchange_slices(th, self.ranges, self.rank, self.group)
        return th

    def check(self) -> None:
        self.eng.check()
        if self.peers is not None and self.eng.status().reserved:
            raise RuntimeError("fused exchange: peer barrier watchdog fired "
                               "(a rank stopped responding)")


class VirtualCluster:
    """All ranks of a sharded run on ONE device, exchanging by device copies.
    Exercises exactly the per-rank layouts/schedules/kernels of the multi-GPU
    path (for bitwise-equality tests without several GPUs)."""

    def __init__(self, dec: Decomposition | None, omega, coupling: float, norm: float | None,
                 world: int, device=None, graphs=None, ranges=None, p2p: bool = False):
        self.ranges = ranges if ranges is not None else partition_rows(dec, world)
        self.ranks = []
        for r in range(world):
            g = (graphs[r] if graphs is not None
                 else DeviceGraph(dec, device=device, row_range=self.ranges[r]))
            e = KuramotoEngine(dec, omega, coupling=coupling, norm=norm, graph=g)
            self.ranks.append((e, workspace_views(e)))
        # fused exchange on one device: every virtual rank's epilogue stores into
        # the others' workspaces (signal-only barrier: ranks run one after another)
        self.peers = None
        if p2p and world > 1:
            bases = [e.workspace.data_ptr() for e, _ in self.ranks]
            offs = [workspace_offsets(e) for e, _ in self.ranks]
            for e, _ in self.ranks:
                zero_peer_counter(e)
            self.peers = [PeerTable(bases, offs, r, self.ranks[r][0].device, False)
                          for r in range(world)]

    @classmethod
    def generated(cls, case, world: int, device=None, smem_budget=None, p2p: bool = False):
        """Every rank of a sharded device-generated graph on one device."""
        from . import gen

        ranges = partition_by_cost(case.offsets(), case.n, case.row_costs(), world)
        graphs = [gen.device_graph(case, device, smem_budget=smem_budget, row_range=rr)[0]
                  for rr in ranges]
        omega, _ = case.state()
        return cls(None, omega, case.coupling, case.n, world, device, graphs, ranges, p2p=p2p)

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
                if self.peers is not None:
                    for (e, _), pt in zip(self.ranks, self.peers):
                        _lib.check(e.lib.cdk_kuramoto_rk4_stage_peers(
                            ctypes.byref(e.graph.struct), e.theta.data_ptr(), e.omega.data_ptr(),
                            e.k_over_n, float(dt), s, e.workspace.data_ptr(),
                            ctypes.byref(pt.struct), None), "rk4_stage_peers")
                        pt.advance(1)
                else:
                    for e, _ in self.ranks:
                        e.rk4_stage(dt, s)
                    self._exchange(s & 1)
            for e, _ in self.ranks:
                _lib.check(e.lib.cdk_kuramoto_advance(ctypes.byref(e.graph.struct),
                                                      e.workspace.data_ptr(), 1, None), "advance")

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
    from bench import (METRIC, UNIT, ClockSampler, _peaks,  # noqa: E402
                       algorithmic_bytes_per_rhs, cfg2_config)

    cfg = getattr(args, "config", "cfg2")
    # fused exchange (NVLink P2P stores + peer barrier) when every peer is
    # reachable; CDK_P2P=0 falls back to the NCCL all-gather after each stage
    from .settings import settings

    p2p = settings().p2p and world > 1 and all(
        torch.cuda.can_device_access_peer(local, q) for q in range(torch.cuda.device_count())
        if q != local)
    if cfg == "cfg5":
        case = gen.config5()
        omega, theta0 = case.state()
        eng = ShardedKuramotoEngine.generated(case, rank, world, p2p=p2p)
        nnz_local = eng.graph.layout.nnz_dir
        workload = ("cfg5 Kuramoto CIA RK4, LFR-style N=8000000 (device-generated, each rank its "
                    "own rows), sharded by community")
        flush = None
    else:
        case = configs.config2()
        dec = case.decomposition()
        omega, theta0 = case.state()
        eng = ShardedKuramotoEngine(dec, omega, case.coupling, case.n, rank, world, p2p=p2p)
        nnz_local = eng.graph.layout.nnz_dir
        workload = "cfg2 Kuramoto CIA RK4, SBM N=200000, sharded by community"
        flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    exchange = eng.verify_fused(theta0, case.dt) if world > 1 else "single rank"
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
            "config": (cfg2_config(case, dec) if cfg != "cfg5" else
                       {"workload": workload, "n_nodes": case.n, "nnz_dir": nnz,
                        "l2": "inputs >> L2"}),
            "setup": {"parallelism": f"community shards x{world}", "exchange": exchange,
                      "ranges": eng.ranges},
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
