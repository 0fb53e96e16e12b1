"""Device-side LFR-style community graph generator (BASELINE config 5, SURVEY
§7.3.1 and §8f rank 1; SPEC.md:61-69,101-109 for the decomposition it feeds).

Config 5 is N = 8e6 nodes and about 1.0e10 directed corrections.  Building
that on the host and shipping ~27 GB of CSR is impractical, so the graph is
generated straight into the stage kernel's layout (csrc/gen.cu, C ABI
``cdk_gen_*``):

* community sizes: power law (exponent 1.5) on [lo, hi], drawn until they
  cover N, then renormalised to sum to N (floor + largest remainders);
* intra: pair {a, b} of community c is MISSING (a -1 correction) iff a
  counter-based hash of (seed, c, min, max) falls below (1 - p_in) * 2^32;
  symmetric, and any row can be regenerated on its own;
* inter: every node gets a propensity d_i = k_out(c_i) * w_i / E[w] with
  k_out(c) = mu/(1-mu) * p_in * (lambda_c - 1) and w ~ truncated Pareto,
  density w^-deg_exp on [1, w_max] (the heavy-tailed degree part);
  n_edges endpoint pairs are drawn by inverse CDF over d (hash of (seed, e, k)),
  pairs inside one community are dropped, duplicates are removed after a
  per-row sort.  n_edges = (sum d / 2) / (1 - sum_c (D_c / D)^2) so the
  expected kept degree is d_i.

Everything is deterministic in (graph_seed, sizes): identical on any GPU
count.  ``oracle/gen.py`` restates the hashes in numpy (test infrastructure).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InputError
from .graph import power_law_sizes
from .plan import (INTER_COST, ROW_COST, HostLayout, _rblocks, community_passes,
                   window_nodes)


@dataclass(frozen=True)
class LfrCase:
    """BASELINE configs[4] family: classical Kuramoto on an LFR-style graph."""

    name: str
    n: int
    size_lo: int
    size_hi: int
    size_exp: float = 1.5
    p_in: float = 0.9
    mu: float = 0.05
    deg_exp: float = 2.5
    w_max: float = 10.0
    coupling: float = 5.0
    dt: float = 0.01
    steps: int = 200
    graph_seed: int = 5001
    state_seed: int = 5101

    def sizes(self) -> np.ndarray:
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([self.graph_seed, 1])))
        a = 1.0 - self.size_exp
        draws = int(2 * self.n / self.size_lo) + 16
        u = rng.random(draws)
        s = (self.size_lo ** a + u * (self.size_hi ** a - self.size_lo ** a)) ** (1.0 / a)
        m = int(np.searchsorted(np.cumsum(s), self.n)) + 1
        rng2 = np.random.Generator(np.random.PCG64(np.random.SeedSequence([self.graph_seed, 2])))
        sizes = power_law_sizes(rng2, m, self.size_exp, float(self.size_lo), float(self.size_hi),
                                self.n)
        if sizes.max() > 0xFFFE:
            raise InputError("community above 65534 nodes")
        return sizes

    def offsets(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.sizes())]).astype(np.int64)

    def propensities(self, offsets: np.ndarray) -> np.ndarray:
        """expected inter degree d_i per node (float64[N])."""
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([self.graph_seed, 3])))
        b = self.deg_exp - 1.0
        u = rng.random(self.n)
        w = (1.0 - u * (1.0 - self.w_max ** -b)) ** (-1.0 / b)
        mean_w = (b / (b - 1.0)) * (1.0 - self.w_max ** (1.0 - b)) / (1.0 - self.w_max ** -b)
        lam = np.diff(offsets).astype(np.float64)
        k_out = self.mu / (1.0 - self.mu) * self.p_in * (lam - 1.0)
        return np.repeat(k_out, np.diff(offsets)) * (w / mean_w)

    def gen_inputs(self):
        """(offsets, node_cdf, n_inter_edges, miss_thr) — the generator's parameters."""
        off = self.offsets()
        d = self.propensities(off)
        D = float(d.sum())
        Dc = np.add.reduceat(d, off[:-1]) if off.shape[0] > 1 else np.zeros(0)
        same = float(((Dc / D) ** 2).sum()) if D > 0 else 0.0
        n_edges = int(round(0.5 * D / max(1.0 - same, 1e-12))) if D > 0 else 0
        cdf = np.cumsum(d) / D if D > 0 else np.linspace(1.0 / self.n, 1.0, self.n)
        cdf[-1] = 1.0
        thr = int(min(round((1.0 - self.p_in) * 2.0 ** 32), 2 ** 32 - 1))
        return off, cdf, n_edges, thr

    def row_costs(self) -> np.ndarray:
        """Expected per-row cost in the planner's model (padded missing-intra
        entries + INTER_COST x expected inter degree + ROW_COST), for sharding."""
        off = self.offsets()
        lam = np.diff(off).astype(np.float64)
        intra = np.repeat(np.ceil((1.0 - self.p_in) * (lam - 1.0) / 8.0) * 8.0, np.diff(off))
        return intra + INTER_COST * self.propensities(off) + ROW_COST

    def state(self):
        """(omega, theta0): omega ~ Cauchy(0, 0.5), theta0 ~ U[0, 2 pi) (BASELINE configs[4])."""
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(self.state_seed)))
        omega = 0.5 * rng.standard_cauchy(self.n)
        theta0 = rng.uniform(0.0, 2.0 * math.pi, self.n)
        return omega, theta0


def config5() -> LfrCase:
    """BASELINE configs[4]: N = 8e6, sizes power law 1.5 on [1e3, 2e4], p_in .9,
    mu .05, degree exponent 2.5, omega ~ Cauchy(0, .5), RK4 dt .01 x 200, K = 5."""
    return LfrCase("cfg5", 8_000_000, 1000, 20000)


def scaled_config5(n: int = 6000, lo: int = 60, hi: int = 900, seed: int = 51) -> LfrCase:
    """Config-5 family at a size the oracle handles."""
    return LfrCase(f"cfg5_n{n}", n, lo, hi, graph_seed=seed, state_seed=seed + 100)


@dataclass
class GeneratedCsr:
    """Device CSR in the layout of plan.build_layout (intra columns community-local)."""

    n_rows: int
    n_comm: int
    comm_off: np.ndarray  # host int64[M+1]
    intra_ptr: np.ndarray  # host int64[N+1] (padded runs)
    inter_ptr: np.ndarray  # host int64[N+1]
    intra_col: object  # device int16 (uint16 bits), +8 slack
    inter_col: object  # device int32, +4 slack
    n_inter_edges: int
    nnz_intra: int
    intra_split: object = None  # device int64 (uint64 bits) or None
    pass_nodes: int = 0
    row_range: tuple | None = None

    def layout(self) -> HostLayout:
        n = self.n_rows
        off = self.comm_off
        rblk_row0, rblk_comm, comm_rblk_off = _rblocks(off, n, self.intra_ptr, self.inter_ptr,
                                                       self.row_range)
        padded = np.diff(self.intra_ptr)
        xcounts = np.diff(self.inter_ptr)
        row_cost = padded.astype(np.float64) + INTER_COST * xcounts + ROW_COST
        split = (self.intra_split.cpu().numpy().view(np.uint64)
                 if self.intra_split is not None else None)
        return HostLayout(n, self.n_comm, off, self.intra_ptr, None, self.inter_ptr, None,
                          rblk_row0, rblk_comm, comm_rblk_off, row_cost,
                          self.nnz_intra, int(self.inter_ptr[-1]), split, self.pass_nodes)

    def split_host(self) -> np.ndarray:
        if self.intra_split is None:
            return np.zeros(self.n_rows, dtype=np.uint64)
        return self.intra_split.cpu().numpy().view(np.uint64)

    def to_host(self):
        """(intra_ptr, intra_col uint16 local, inter_ptr, inter_col int32) on the host."""
        ni, nx = int(self.intra_ptr[-1]), int(self.inter_ptr[-1])
        return (self.intra_ptr, self.intra_col[:ni].cpu().numpy().view(np.uint16),
                self.inter_ptr, self.inter_col[:nx].cpu().numpy())


def generate(case: LfrCase, device=None, stream=None, pass_nodes: int | None = None,
             row_range=None) -> GeneratedCsr:
    """Run the device generator for ``case``; returns the CSR on ``device``.
    Rows of communities wider than ``pass_nodes`` (default: the stage
    kernel's window) get one sub-run per window pass (cdk_graph.intra_split).
    ``row_range=(lo, hi)``: generate only those rows (a rank's shard, cut at
    community boundaries); other rows are empty, columns stay global, and the
    shard's rows are identical to the same rows of the full graph."""
    import torch

    pass_nodes = window_nodes() if pass_nodes is None else int(pass_nodes)
    lo, hi = (0, case.n) if row_range is None else (int(row_range[0]), int(row_range[1]))
    dev = torch.device(device if device is not None else "cuda")
    lib = _lib.lib()
    off, cdf, n_edges, thr = case.gen_inputs()
    n, m = case.n, off.shape[0] - 1
    d_off = torch.from_numpy(off).to(dev)
    d_cdf = torch.from_numpy(cdf).to(dev)
    p = _lib.CdkGenParams(seed=int(case.graph_seed), n_rows=n, n_comm=m,
                          comm_off=d_off.data_ptr(), node_cdf=d_cdf.data_ptr(),
                          n_inter_edges=n_edges, miss_thr=thr, pass_nodes=pass_nodes,
                          row_lo=lo, row_hi=hi)
    pp = ctypes.byref(p)
    sp = _lib.stream_ptr(stream)

    # intra: padded run lengths (per-pass sub-runs) -> pointers -> columns
    cnt = torch.zeros(n, dtype=torch.int64, device=dev)
    raw = torch.zeros(n, dtype=torch.int64, device=dev)
    split = torch.zeros(n, dtype=torch.int64, device=dev)
    _lib.check(lib.cdk_gen_intra_count(pp, cnt.data_ptr(), raw.data_ptr(), split.data_ptr(), sp),
               "gen_intra_count")
    nnz_intra = int(raw.sum().item())
    del raw
    iptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(cnt, 0, out=iptr[1:])
    ni = int(iptr[-1].item())
    icol = torch.full((ni + 8,), -1, dtype=torch.int16, device=dev)
    _lib.check(lib.cdk_gen_intra_fill(pp, iptr.data_ptr(), split.data_ptr(), icol.data_ptr(), sp),
               "gen_intra_fill")
    if not (community_passes(off, pass_nodes) > 1).any():
        split = None

    # inter: counts -> scatter -> per-row sort + dedupe -> compact
    cnt.zero_()
    _lib.check(lib.cdk_gen_inter_count(pp, cnt.data_ptr(), sp), "gen_inter_count")
    rptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(cnt, 0, out=rptr[1:])
    nraw = int(rptr[-1].item())
    raw = torch.empty(max(nraw, 1), dtype=torch.int32, device=dev)
    cursor = rptr[:-1].clone()
    _lib.check(lib.cdk_gen_inter_fill(pp, cursor.data_ptr(), raw.data_ptr(), sp), "gen_inter_fill")
    del cursor
    uniq = cnt
    _lib.check(lib.cdk_gen_inter_sort(n, rptr.data_ptr(), raw.data_ptr(), uniq.data_ptr(), sp),
               "gen_inter_sort")
    xptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(uniq, 0, out=xptr[1:])
    nx = int(xptr[-1].item())
    xcol = torch.zeros(nx + 4, dtype=torch.int32, device=dev)
    _lib.check(lib.cdk_gen_inter_compact(n, rptr.data_ptr(), xptr.data_ptr(), raw.data_ptr(),
                                         xcol.data_ptr(), sp), "gen_inter_compact")
    del raw
    return GeneratedCsr(n, m, off, iptr.cpu().numpy(), xptr.cpu().numpy(), icol, xcol, n_edges,
                        nnz_intra, split, pass_nodes, None if row_range is None else (lo, hi))


def device_graph(case: LfrCase, device=None, sm_count: int | None = None,
                 smem_budget: int | None = None, row_range=None):
    """(DeviceGraph, GeneratedCsr) for ``case``: generate, plan, rebase in place.
    ``smem_budget`` shrinks the stage kernel's window (tests: multi-pass paths
    at small sizes); ``row_range`` generates one rank's shard."""
    from .plan import ROWS_CAP, SMEM_BUDGET, DeviceGraph

    budget = SMEM_BUDGET if smem_budget is None else int(smem_budget)
    csr = generate(case, device, pass_nodes=window_nodes(ROWS_CAP, budget), row_range=row_range)
    dg = DeviceGraph.from_device_csr(csr.layout(), csr.intra_col, csr.inter_col,
                                     csr.intra_col.device, sm_count=sm_count,
                                     split_dev=csr.intra_split, smem_budget=budget,
                                     row_range=row_range)
    csr.intra_col = None  # rebased + bank-ordered copy lives in dg (the original is freed)
    return dg, csr


__all__ = ["LfrCase", "config5", "scaled_config5", "GeneratedCsr", "generate", "device_graph"]
