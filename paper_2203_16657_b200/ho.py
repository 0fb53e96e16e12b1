"""Higher-order (triadic) Kuramoto on the 3-cliques of a community graph
(BASELINE config 3) — model, host preparation and the
device engine (csrc/ho.cu, C ABI ``cdk_ho_*``).

    theta'_i = omega_i + (K1/N) sum_j a_ij sin(theta_j - theta_i)
             + (K2/N^2) sum_{(j,k) ordered, {i,j,k} triangle} sin(theta_j + theta_k - 2 theta_i)

Host preparation (once per decomposition):
* the proper missing-edge graph inside communities (S entries with sign -1,
  diagonal dropped) as a CSR with global columns;
* its triangles (native ``cdk_host_triangles``) -> per-row pairs (j, k);
* triangles spanning communities / the NONE pool: every such triangle has a
  vertex with two inter-community edges in it, so it is found by checking the
  pairs of inter neighbours of every node -> per-row pairs flagged j < 0.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import BlowUpError, InputError
from .graph import NONE, Decomposition
from .plan import build_layout


@dataclass(frozen=True)
class HigherOrderKuramoto:
    omega: np.ndarray
    k1: float = 1.0
    k2: float = 0.5
    norm: float | None = None
    state_space: str = "circle"

    def n(self) -> int:
        return int(np.asarray(self.omega).shape[0])

    def norm_value(self) -> float:
        return float(self.norm if self.norm is not None else self.n())


def ho_kuramoto_model(omega, k1=1.0, k2=0.5, norm=None) -> HigherOrderKuramoto:
    return HigherOrderKuramoto(np.asarray(omega, dtype=np.float64), float(k1), float(k2), norm)


def _csr(rows, cols, n):
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=ptr[1:])
    return ptr, cols.astype(np.int32)


def missing_csr(dec: Decomposition):
    rows, cols, sg = dec.directed()
    m = sg < 0
    return _csr(rows[m], cols[m], dec.n_nodes)


def inter_csr(dec: Decomposition):
    rows, cols, sg = dec.directed()
    m = sg > 0
    return _csr(rows[m], cols[m], dec.n_nodes)


def missing_triangles(dec: Decomposition) -> np.ndarray:
    """Triangles {i<j<k} of the missing-edge graph (int32 [T, 3])."""
    ptr, col = missing_csr(dec)
    lib = _lib.load_library()
    n = dec.n_nodes
    P = ctypes.c_void_p
    cnt = lib.cdk_host_triangles(ptr.ctypes.data_as(P), col.ctypes.data_as(P), n, None, 0)
    if cnt < 0:
        raise InputError("cdk_host_triangles failed")
    out = np.empty((max(cnt, 1), 3), dtype=np.int32)
    lib.cdk_host_triangles(ptr.ctypes.data_as(P), col.ctypes.data_as(P), n,
                           out.ctypes.data_as(P), cnt)
    return out[:cnt]


def spanning_triangles(dec: Decomposition) -> np.ndarray:
    """Triangles of the graph that are not inside one community (int64 [T, 3])."""
    n = dec.n_nodes
    comm = dec.partition.comm_of_permuted()
    iptr, icol = inter_csr(dec)
    s = dec.correction
    miss = s.sgn < 0
    missing = set(zip(s.iu[miss & (s.iu != s.iv)].tolist(), s.iv[miss & (s.iu != s.iv)].tolist()))
    xu, xv = s.iu[~miss], s.iv[~miss]
    inter = set(zip(xu.tolist(), xv.tolist()))

    def edge(a, b):
        if a > b:
            a, b = b, a
        if comm[a] == comm[b] and comm[a] != NONE:
            return (a, b) not in missing
        return (a, b) in inter

    found = set()
    deg = np.diff(iptr)
    for w in np.nonzero(deg >= 2)[0].tolist():
        nb = icol[iptr[w]: iptr[w + 1]].tolist()
        for p in range(len(nb)):
            for q in range(p + 1, len(nb)):
                if edge(nb[p], nb[q]):
                    found.add(tuple(sorted((w, nb[p], nb[q]))))
    if not found:
        return np.zeros((0, 3), dtype=np.int64)
    return np.array(sorted(found), dtype=np.int64)


def triangle_pairs(n: int, miss_tri: np.ndarray, span_tri: np.ndarray):
    """Per-row (j, k) pairs: missing-graph triangles as (j, k), spanning ones
    as (-j-1, k).  CSR by row."""
    rows, js, ks = [], [], []
    for tri, flag in ((np.asarray(miss_tri, np.int64), False),
                      (np.asarray(span_tri, np.int64), True)):
        if tri.size == 0:
            continue
        for a, b, c in ((0, 1, 2), (1, 0, 2), (2, 0, 1)):
            rows.append(tri[:, a])
            js.append(-tri[:, b] - 1 if flag else tri[:, b])
            ks.append(tri[:, c])
    if not rows:
        return np.zeros(n + 1, np.int64), np.zeros((1, 2), np.int32)
    r = np.concatenate(rows)
    jk = np.stack([np.concatenate(js), np.concatenate(ks)], 1)
    order = np.argsort(r, kind="stable")
    r, jk = r[order], jk[order]
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=ptr[1:])
    return ptr, jk.astype(np.int32)


class HoDeviceGraph:
    def __init__(self, dec: Decomposition, device=None):
        import torch

        dev = torch.device(device if device is not None else "cuda")
        n = dec.n_nodes
        lay = build_layout(dec)
        mptr, mcol = missing_csr(dec)
        xptr, xcol = inter_csr(dec)
        self.miss_tri = missing_triangles(dec)
        self.span_tri = spanning_triangles(dec)
        tptr, tjk = triangle_pairs(n, self.miss_tri, self.span_tri)
        self.tri_pairs = int(tptr[-1])  # triangle incidences one RHS evaluates

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

        self._t = {
            "rblk_row0": up(lay.rblk_row0), "rblk_comm": up(lay.rblk_comm),
            "comm_rblk_off": up(lay.comm_rblk_off),
            "miss_ptr": up(mptr), "miss_col": up(mcol if mcol.size else np.zeros(1, np.int32)),
            "inter_ptr": up(xptr), "inter_col": up(xcol if xcol.size else np.zeros(1, np.int32)),
            "tri_ptr": up(tptr), "tri_jk": up(tjk),
        }
        t = self._t
        self.n_rows = n
        self.device = dev
        self.struct = _lib.CdkHoGraph(
            n_rows=n, n_rblk=lay.n_rblk, n_comm=lay.n_comm,
            rblk_row0=t["rblk_row0"].data_ptr(), rblk_comm=t["rblk_comm"].data_ptr(),
            comm_rblk_off=t["comm_rblk_off"].data_ptr(), miss_ptr=t["miss_ptr"].data_ptr(),
            miss_col=t["miss_col"].data_ptr(), inter_ptr=t["inter_ptr"].data_ptr(),
            inter_col=t["inter_col"].data_ptr(), tri_ptr=t["tri_ptr"].data_ptr(),
            tri_jk=t["tri_jk"].data_ptr())


class HOEngine:
    """Device-resident triadic Kuramoto CIA engine (permuted order)."""

    def __init__(self, dec: Decomposition, omega, k1: float, k2: float, norm=None, device=None,
                 graph: HoDeviceGraph | None = None):
        import torch

        self.lib = _lib.lib()
        self.graph = graph if graph is not None else HoDeviceGraph(dec, device)
        self.device = self.graph.device
        n = self.graph.n_rows
        self.n = n
        norm = float(norm if norm is not None else n)
        self.k1n = float(k1) / norm
        self.k2n2 = float(k2) / norm**2
        self.omega = torch.as_tensor(np.asarray(omega, np.float64)).to(self.device)
        self.theta = torch.zeros(n, dtype=torch.float64, device=self.device)
        nb = int(self.lib.cdk_ho_workspace_bytes(ctypes.byref(self.graph.struct)))
        self.workspace = torch.empty(max(nb, 256), dtype=torch.uint8, device=self.device)
        self._gp = ctypes.byref(self.graph.struct)
        self._rhs_ws = None

    def set_state(self, theta, stream=None):
        import torch

        t = theta if torch.is_tensor(theta) else torch.from_numpy(np.ascontiguousarray(theta,
                                                                                   np.float64))
        self.theta.copy_(t.to(self.device, torch.float64))
        _lib.check(self.lib.cdk_ho_prepare(self._gp, self.theta.data_ptr(),
                                           self.workspace.data_ptr(), _lib.stream_ptr(stream)),
                   "ho_prepare")

    def rhs(self, theta, stream=None):
        import torch

        th = torch.as_tensor(theta, dtype=torch.float64).to(self.device).contiguous()
        out = torch.empty(self.n, dtype=torch.float64, device=self.device)
        if self._rhs_ws is None:
            self._rhs_ws = torch.empty_like(self.workspace)
        _lib.check(self.lib.cdk_ho_rhs(self._gp, th.data_ptr(), self.omega.data_ptr(), self.k1n,
                                       self.k2n2, out.data_ptr(), self._rhs_ws.data_ptr(),
                                       _lib.stream_ptr(stream)), "ho_rhs")
        return out

    def rk4(self, dt: float, n_steps: int, stream=None):
        _lib.check(self.lib.cdk_ho_rk4(self._gp, self.theta.data_ptr(), self.omega.data_ptr(),
                                       self.k1n, self.k2n2, float(dt), int(n_steps),
                                       self.workspace.data_ptr(), _lib.stream_ptr(stream)),
                   "ho_rk4")

    def check(self, stream=None):
        st = _lib.CdkRunStatus()
        _lib.check(self.lib.cdk_ho_status(self._gp, self.workspace.data_ptr(), ctypes.byref(st),
                                          _lib.stream_ptr(stream)), "ho_status")
        if st.nonfinite:
            raise BlowUpError(int(st.first_bad_step))
