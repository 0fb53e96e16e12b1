"""Cucker–Smale flocking in 2-D with a per-community polynomial expansion
(BASELINE config 4) — model, P2 fit, host plan and the
device engine (csrc/cs.cu, C ABI ``cdk_cs_*``).

    s_m' = v_m
    v_m' = (1/N) sum_l a_ml eta(|s_l - s_m|^2) (v_l - v_m),  eta(y) = K / (sigma^2 + y)^beta

CIA (PAPER.md:653-703 structure, polynomial basis instead of Fourier as the
config asks): for community c with centre mu_c and scale L_c, scaled
positions p = (s - mu_c)/L_c, u = |p_l - p_m|^2 and the fitted
eta(L_c^2 u) ~ sum_{k<=8} chat_k u^k.  Expanding u^k binomially,

    sum_{l in c} eta_lm f_l = sum_{p+q<=16} H^f_{pq} x_m^p y_m^q,
    H^f = T_c M^f,   M^f_{ij} = sum_{l in c} x_l^i y_l^j f_l   (f in {1, v_x, v_y}),

with T_c[pq, ij] = chat_{a+b} C(a+b, a) C(2a, i) C(2b, j) (-1)^{p+q} for
a = (p+i)/2, b = (q+j)/2 integer, a+b <= 8.  The dense part is
(1/N)(G^v - v_m G^1); the sparse correction uses the EXACT eta.
Fit: least squares in the monomials u^k on 2(p+1) Chebyshev
nodes of [0, 4].  Domain: |p| <= 1 for every node over the whole trajectory
(mu_c, L_c chosen from the initial state and the largest speed); a node that
leaves it raises DomainViolationError.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from math import comb

import numpy as np

from . import _lib
from .errors import BlowUpError, DomainViolationError, InputError
from .graph import Decomposition
from .settings import settings
from .plan import build_layout

DEG = 8
D2 = 2 * DEG
NMON = (D2 + 1) * (D2 + 2) // 2  # 153 monomials x^i y^j, i + j <= 16


def mono_index():
    """(i, j) of the packed monomial index, i + j <= 16 (i-major)."""
    return [(i, j) for i in range(D2 + 1) for j in range(D2 + 1 - i)]


@dataclass(frozen=True)
class CuckerSmale:
    K: float = 1.0
    sigma: float = 1.0
    beta: float = 0.25
    norm: float | None = None
    degree: int = DEG

    def eta(self, y):
        return self.K / (self.sigma**2 + np.asarray(y)) ** self.beta


def fit_eta(model: CuckerSmale, L: float, deg: int = DEG):
    """Least-squares fit of eta(L^2 u) on u in [0, 4] in the monomials u^k,
    on 2(deg+1) Chebyshev nodes.  Returns (chat[deg+1], sup_err)."""
    m = 2 * (deg + 1)
    nodes = 2.0 + 2.0 * np.cos((2 * np.arange(m) + 1) * np.pi / (2 * m))
    V = np.vander(nodes, deg + 1, increasing=True)
    c, *_ = np.linalg.lstsq(V, model.eta(L * L * nodes), rcond=None)
    grid = np.linspace(0.0, 4.0, 2001)
    sup = float(np.abs(np.vander(grid, deg + 1, increasing=True) @ c - model.eta(L * L * grid)).max())
    return c, sup


_BASIS = None


def _contraction_basis() -> np.ndarray:
    """B[k, pq, ij] = C(k,a) C(2a,i) C(2b,j) (-1)^{p+q} for a+b = k (else 0)."""
    global _BASIS
    if _BASIS is None:
        mon = mono_index()
        B = np.zeros((DEG + 1, NMON, NMON))
        for r, (p, q) in enumerate(mon):
            for s_, (i, j) in enumerate(mon):
                if (p + i) % 2 or (q + j) % 2:
                    continue
                a, b = (p + i) // 2, (q + j) // 2
                k = a + b
                if k > DEG or i > 2 * a or j > 2 * b:
                    continue
                B[k, r, s_] = comb(k, a) * comb(2 * a, i) * comb(2 * b, j) * (-1) ** (p + q)
        _BASIS = B
    return _BASIS


def contraction_pattern():
    """The shared sparsity of T_c (module docstring): for output monomial r the
    nonzero inputs s with their degree k(r, s) and coefficient B[k, r, s].
    CSR by r: (t_ptr int32[NMON+1], t_col int32 = s | k << 8, t_coef f64);
    T_c[r, s] = chat_c[k] * t_coef exactly as contraction_tensor forms it."""
    B = _contraction_basis()
    nz = B != 0
    if np.any(nz.sum(axis=0) > 1):
        raise AssertionError("contraction basis: more than one degree per (r, s)")
    k_of = np.argmax(nz, axis=0)  # [r, s]
    any_nz = nz.any(axis=0)
    ptr = np.zeros(NMON + 1, dtype=np.int32)
    ptr[1:] = np.cumsum(any_nz.sum(axis=1))
    r_idx, s_idx = np.nonzero(any_nz)  # row-major: r ascending, s ascending
    k = k_of[r_idx, s_idx]
    col = (s_idx | (k << 8)).astype(np.int32)
    coef = B[k, r_idx, s_idx]
    return ptr, col, coef


def contraction_tensor(chat) -> np.ndarray:
    """T[pq, ij] of the module docstring (NMON x NMON)."""
    return np.tensordot(np.asarray(chat, np.float64), _contraction_basis(), axes=(0, 0))


@dataclass
class CsPlan:
    mu: np.ndarray  # [M, 2]
    L: np.ndarray  # [M]
    chat: np.ndarray  # [M, DEG+1]
    T: np.ndarray  # [M, NMON, NMON]
    sup_err: np.ndarray  # [M]


def cs_plan(model: CuckerSmale, dec: Decomposition, pos0, vel0, t_end: float,
            margin: float = 1.05) -> CsPlan:
    """Per-community centre/scale and P2 fit covering the whole trajectory:
    L_c = (max_l |s_l - mu_c| + t_end * max_l |v_l|) * margin, so |p| <= 1
    while every speed stays below the initial maximum (CS dynamics do not
    increase max |v|: velocities relax toward weighted averages)."""
    off = dec.offsets
    m = dec.partition.n_comm
    pos0 = np.asarray(pos0, np.float64)
    vel0 = np.asarray(vel0, np.float64)
    mu = np.zeros((m, 2))
    L = np.zeros(m)
    chat = np.zeros((m, DEG + 1))
    T = np.zeros((m, NMON, NMON))
    sup = np.zeros(m)
    vmax = float(np.sqrt((vel0 ** 2).sum(1)).max()) if vel0.size else 0.0
    for c in range(m):
        s = pos0[off[c]: off[c + 1]]
        mu[c] = s.mean(0)
        r0 = float(np.sqrt(((s - mu[c]) ** 2).sum(1)).max())
        L[c] = max((r0 + t_end * vmax) * margin, 1e-6)
        chat[c], sup[c] = fit_eta(model, L[c])
        T[c] = contraction_tensor(chat[c])
    return CsPlan(mu, L, chat, T, sup)


def _csr(rows, cols, n):
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=ptr[1:])
    return ptr, cols.astype(np.int32)


def _csr_bank_spread(rows, cols, n, base_of_row, parity_of_row):
    """CSR of the missing intra edges with every row's entries ordered for the
    shared-memory window of cs_sparse_win_kernel: a quarter-warp is two
    consecutive rows x 4 lanes reading 4 consecutive entries each, 16 bytes
    per lane, so its 8 loads are conflict-free iff their window indices differ
    mod 8.  The even row of a pair lists its entries of bank groups 0-3 first
    and 4-7 second, the odd row the other way round, and inside a half the
    entries go round-robin over the half's four groups.  (Random order costs
    ~2.3 wavefronts per ideal one.)  Any fixed order is a valid summation
    order; both sparse kernels read the same one."""
    j = cols - base_of_row[rows]
    g = j & 7
    first = np.lexsort((cols, g, rows))
    r_s, g_s = rows[first], g[first]
    key = r_s * 8 + g_s
    start = np.r_[True, key[1:] != key[:-1]]
    idx = np.arange(key.shape[0])
    rank = idx - np.maximum.accumulate(np.where(start, idx, 0))
    half = (g_s >> 2) ^ parity_of_row[r_s]
    order = np.lexsort((g_s & 3, rank, half, r_s))
    rows_o, cols_o = r_s[order], cols[first][order]
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows_o, minlength=n), out=ptr[1:])
    return ptr, cols_o.astype(np.int32)


class CsDeviceGraph:
    def __init__(self, dec: Decomposition, plan: CsPlan, device=None):
        import torch

        dev = torch.device(device if device is not None else "cuda")
        n = dec.n_nodes
        lay = build_layout(dec)
        rows, cols, sg = dec.directed()
        if settings().cs_bank_spread:
            comm = dec.partition.comm_of_permuted()
            base = np.where(comm >= 0, dec.offsets[np.maximum(comm, 0)], 0).astype(np.int64)
            rb_of_row = np.searchsorted(lay.rblk_row0, np.arange(n), side="right") - 1
            parity = ((np.arange(n) - lay.rblk_row0[np.minimum(rb_of_row, lay.n_rblk - 1)]) & 1
                      ).astype(np.int64)
            mptr, mcol = _csr_bank_spread(rows[sg < 0], cols[sg < 0], n, base, parity)
        else:
            mptr, mcol = _csr(rows[sg < 0], cols[sg < 0], n)
        xptr, xcol = _csr(rows[sg > 0], cols[sg > 0], n)

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

        self._t = {
            "comm_off": up(dec.offsets),
            "rblk_row0": up(lay.rblk_row0), "rblk_comm": up(lay.rblk_comm),
            "miss_ptr": up(mptr), "miss_col": up(mcol if mcol.size else np.zeros(1, np.int32)),
            "inter_ptr": up(xptr), "inter_col": up(xcol if xcol.size else np.zeros(1, np.int32)),
            "mu": up(plan.mu), "inv_L": up(1.0 / plan.L), "chat": up(plan.chat),
        }
        tp, tc, tcoef = contraction_pattern()
        self._t.update(t_ptr=up(tp), t_col=up(tc), t_coef=up(tcoef))
        t = self._t
        self.n_rows = n
        self.n_comm = dec.partition.n_comm
        self.device = dev
        self.plan = plan
        self.struct = _lib.CdkCsGraph(
            n_rows=n, n_comm=self.n_comm, n_rblk=lay.n_rblk,
            max_comm=int(np.diff(dec.offsets).max()) if self.n_comm else 0,
            comm_off=t["comm_off"].data_ptr(), rblk_row0=t["rblk_row0"].data_ptr(),
            rblk_comm=t["rblk_comm"].data_ptr(), miss_ptr=t["miss_ptr"].data_ptr(),
            miss_col=t["miss_col"].data_ptr(), inter_ptr=t["inter_ptr"].data_ptr(),
            inter_col=t["inter_col"].data_ptr(), mu=t["mu"].data_ptr(),
            inv_L=t["inv_L"].data_ptr(), chat=t["chat"].data_ptr(),
            t_ptr=t["t_ptr"].data_ptr(), t_col=t["t_col"].data_ptr(),
            t_coef=t["t_coef"].data_ptr())


class CSEngine:
    """Device-resident Cucker–Smale CIA engine (permuted order, 2-D)."""

    def __init__(self, dec: Decomposition, model: CuckerSmale, pos0, vel0, t_end: float,
                 device=None, plan: CsPlan | None = None):
        import torch

        self.lib = _lib.lib()
        self.model = model
        self.plan = plan if plan is not None else cs_plan(model, dec, pos0, vel0, t_end)
        self.graph = CsDeviceGraph(dec, self.plan, device)
        self.device = self.graph.device
        n = self.graph.n_rows
        self.n = n
        self.inv_n = 1.0 / float(model.norm if model.norm is not None else n)
        self.pos = torch.zeros((n, 2), dtype=torch.float64, device=self.device)
        self.vel = torch.zeros((n, 2), dtype=torch.float64, device=self.device)
        nb = int(self.lib.cdk_cs_workspace_bytes(ctypes.byref(self.graph.struct)))
        self.workspace = torch.empty(max(nb, 256), dtype=torch.uint8, device=self.device)
        self._gp = ctypes.byref(self.graph.struct)
        self.set_state(pos0, vel0)

    def _params(self):
        m = self.model
        return (float(m.K), float(m.sigma) ** 2, float(m.beta), self.inv_n)

    def set_state(self, pos, vel, stream=None):
        import torch

        self.pos.copy_(torch.as_tensor(np.asarray(pos, np.float64)).to(self.device))
        self.vel.copy_(torch.as_tensor(np.asarray(vel, np.float64)).to(self.device))
        _lib.check(self.lib.cdk_cs_prepare(self._gp, self.workspace.data_ptr(),
                                           _lib.stream_ptr(stream)), "cs_prepare")

    def rhs(self, pos, vel, stream=None):
        """(s', v') at (pos, vel): s' = vel, v' from the CIA kernels."""
        import torch

        p = torch.as_tensor(np.asarray(pos, np.float64)).to(self.device).contiguous()
        v = torch.as_tensor(np.asarray(vel, np.float64)).to(self.device).contiguous()
        out = torch.empty((self.n, 2), dtype=torch.float64, device=self.device)
        K, s2, beta, inv_n = self._params()
        _lib.check(self.lib.cdk_cs_rhs(self._gp, p.data_ptr(), v.data_ptr(), K, s2, beta, inv_n,
                                       out.data_ptr(), self.workspace.data_ptr(),
                                       _lib.stream_ptr(stream)), "cs_rhs")
        self.check_domain()
        return v.clone(), out

    def rk4(self, dt: float, n_steps: int, stream=None):
        K, s2, beta, inv_n = self._params()
        _lib.check(self.lib.cdk_cs_rk4(self._gp, self.pos.data_ptr(), self.vel.data_ptr(), K, s2,
                                       beta, inv_n, float(dt), int(n_steps),
                                       self.workspace.data_ptr(), _lib.stream_ptr(stream)),
                   "cs_rk4")

    def status(self, stream=None):
        st = _lib.CdkRunStatus()
        _lib.check(self.lib.cdk_cs_status(self._gp, self.workspace.data_ptr(), ctypes.byref(st),
                                          _lib.stream_ptr(stream)), "cs_status")
        return st

    def check_domain(self):
        st = self.status()
        if st.reserved:
            raise DomainViolationError(f"{st.reserved} node-stages left the expansion domain")

    def check(self):
        st = self.status()
        if st.nonfinite:
            raise BlowUpError(int(st.first_bad_step))
        if st.reserved:
            raise DomainViolationError(f"{st.reserved} node-stages left the expansion domain")


__all__ = ["CuckerSmale", "fit_eta", "contraction_tensor", "cs_plan", "CsPlan", "CSEngine",
           "mono_index", "NMON", "DEG", "InputError"]
