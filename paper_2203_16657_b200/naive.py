"""Direct-sum (naive-mode) right-hand sides on the device — the paper's
accuracy check and the SPEC's ``rhs mode = naive`` (SPEC.md:368-374,
472-474).

The direct sum walks the FULL edge list of the graph (D + S reconstructed,
``Decomposition.graph()``) with the exact coupling, through the device twins
of the reference kernels — the same realisation SURVEY §3.2 measured
(``pairs_trig``/``pairs_cs`` with sgn = +1):

* Kuramoto           out = omega + K/N sum_{(u,v) in E} sin(x_v - x_u) (both ends)
                     -> cdk_pairs_trig, d_sin = (0, K); higher harmonics: the
                     model's d_cos/d_sin (p harmonics, exact h)
* higher-order       + 2 K2/N^2 sum_{triangles {a,b,c}} sin(x_b + x_c - 2 x_a) (+ rotations)
                     -> cdk_pairs_trig (K1) + cdk_triangles_sin
* Cucker-Smale       s' = v, v' = (1/N) sum_{(u,v)} eta(|s_v - s_u|^2) (v_v - v_u) (both ends)
                     -> cdk_pairs_cs (exact eta, sgn = +1)

``NaiveEngine`` keeps the edge list (and triangles) on the device; RK4/Euler
combine the stages with device tensor arithmetic in the oracle's order
(oracle/cia.py).  Kernel-evaluation counts (the complexity
witness): 2|E| per RHS (+ 6 T for the triadic term: 3 vertices x 2 orders).
Memory guard: N > 2^15 raises MemoryGuardError.
"""

from __future__ import annotations

import math

import numpy as np

from . import _kernels, _lib
from .errors import InputError, MemoryGuardError
from .graph import Graph

NAIVE_N_CAP = 2**15
TWO_PI = 2.0 * math.pi


def triangles(graph: Graph) -> np.ndarray:
    """All 3-cliques {a < b < c} of an undirected graph, int64 [T, 3]."""
    n = graph.n_nodes
    e = graph.edges
    if e.shape[0] == 0:
        return np.zeros((0, 3), np.int64)
    order = np.lexsort((e[:, 1], e[:, 0]))
    u, v = e[order, 0], e[order, 1]
    ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(u, minlength=n), out=ptr[1:])
    out = []
    for a in range(n):
        na = v[ptr[a]:ptr[a + 1]]  # neighbours > a, sorted
        for b in na.tolist():
            nb = v[ptr[b]:ptr[b + 1]]  # neighbours > b
            c = np.intersect1d(na, nb, assume_unique=True)
            if c.size:
                out.append(np.stack([np.full(c.size, a), np.full(c.size, b), c], 1))
    return np.concatenate(out).astype(np.int64) if out else np.zeros((0, 3), np.int64)


def _wrap(x):
    """(-pi, pi], same formula as the CUDA epilogue and oracle/cia.py."""
    import torch

    return x - TWO_PI * torch.ceil((x - math.pi) / TWO_PI)


class NaiveEngine:
    """Direct-sum RHS of ``model`` over ``graph`` (node order = the state's)."""

    def __init__(self, model, graph: Graph, device=None):
        import torch

        from .cs import CuckerSmale
        from .harmonics import HigherHarmonicsKuramoto
        from .ho import HigherOrderKuramoto
        from .models import Kuramoto

        if graph.n_nodes > NAIVE_N_CAP:
            raise MemoryGuardError(f"naive mode refuses N = {graph.n_nodes} > {NAIVE_N_CAP} "
                                   "(O(N^2) edge list; SPEC.md:614)")
        _lib.lib()
        self.device = torch.device(device if device is not None else "cuda")
        self.model = model
        self.n = graph.n_nodes
        e = graph.edges
        self.iu = torch.as_tensor(e[:, 0].copy(), dtype=torch.int64, device=self.device)
        self.iv = torch.as_tensor(e[:, 1].copy(), dtype=torch.int64, device=self.device)
        self.sgn = torch.ones(e.shape[0], dtype=torch.float64, device=self.device)
        self.n_edges = int(e.shape[0])
        self.tri = None
        self.n_tri = 0
        if isinstance(model, (Kuramoto, HigherOrderKuramoto, HigherHarmonicsKuramoto)):
            self.kind = "ho" if isinstance(model, HigherOrderKuramoto) else "kuramoto"
            if model.n() != self.n:
                raise InputError("omega shape does not match the graph")
            self.omega = torch.as_tensor(np.asarray(model.omega, np.float64), device=self.device)
            self.norm = model.norm_value()
            if isinstance(model, HigherHarmonicsKuramoto):  # h = p harmonics
                self.d_cos = torch.as_tensor(np.asarray(model.d_cos, np.float64),
                                             device=self.device)
                self.d_sin = torch.as_tensor(np.asarray(model.d_sin, np.float64),
                                             device=self.device)
            else:
                k1 = model.coupling if self.kind == "kuramoto" else model.k1
                self.d_cos = torch.zeros(2, dtype=torch.float64, device=self.device)
                self.d_sin = torch.tensor([0.0, float(k1)], dtype=torch.float64,
                                          device=self.device)
            if self.kind == "ho":
                t = triangles(graph)
                self.n_tri = int(t.shape[0])
                self.tri = torch.as_tensor(t, device=self.device)
                self.k2_coef = 2.0 * float(model.k2) / self.norm**2
        elif isinstance(model, CuckerSmale):
            self.kind = "cs"
            self.norm = float(model.norm if model.norm is not None else self.n)
        else:
            raise InputError(f"naive mode: unsupported model {type(model).__name__}")

    @property
    def kernel_evals_per_rhs(self) -> int:
        return 2 * self.n_edges + 6 * self.n_tri

    def rhs(self, x):
        """Direct-sum derivative of the device state ``x`` ([N] or [N, 4])."""
        import torch

        x = torch.as_tensor(x, dtype=torch.float64).to(self.device).contiguous()
        if self.kind == "cs":
            pos, vel = x[:, :2].contiguous(), x[:, 2:].contiguous()
            acc = torch.zeros_like(vel)
            m = self.model
            _kernels.pairs_cs(self.iu, self.iv, pos, vel, 1.0 / self.norm, m.K, m.sigma**2,
                              m.beta, self.sgn, acc)
            return torch.cat([vel, acc], 1)
        out = self.omega.clone()
        _kernels.pairs_trig(self.iu, self.iv, x, 1.0 / self.norm, self.d_cos, self.d_sin, math.pi,
                            self.sgn, out)
        if self.n_tri:
            L = _lib.lib()
            _lib.check(L.cdk_triangles_sin(self.tri.data_ptr(), self.n_tri, x.data_ptr(),
                                           self.k2_coef, out.data_ptr(), _lib.stream_ptr()),
                       "triangles_sin")
        return out

    def _finish_step(self, x, step: int):
        import torch

        from .errors import BlowUpError

        if self.kind != "cs":
            x = _wrap(x)
        if not bool(torch.isfinite(x).all()):
            raise BlowUpError(step)
        return x

    def rk4(self, x, dt: float, n_steps: int, step0: int = 0):
        """Classical RK4 in the oracle's arithmetic order (oracle/cia.py:82-102)."""
        import torch

        x = torch.as_tensor(x, dtype=torch.float64).to(self.device).clone()
        h2, h6 = dt / 2.0, dt / 6.0
        for s in range(1, n_steps + 1):
            k1 = self.rhs(x)
            k2 = self.rhs(x + h2 * k1)
            k3 = self.rhs(x + h2 * k2)
            k4 = self.rhs(x + dt * k3)
            x = x + h6 * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
            x = self._finish_step(x, step0 + s)
        return x

    def euler(self, x, dt: float, n_steps: int, step0: int = 0):
        import torch

        x = torch.as_tensor(x, dtype=torch.float64).to(self.device).clone()
        for s in range(1, n_steps + 1):
            x = x + dt * self.rhs(x)
            x = self._finish_step(x, step0 + s)
        return x
