"""The remaining model paths of SURVEY §8(f) rank 4 on the device, composed
of the kernel twins (no new orchestration semantics):

* ``DesaiZwanzig`` (PAPER §A.4): x' = -V'(x) + (1/N) sum_l a_ml
  h(x_l - x_m) with a polynomial difference coupling h (default h(x) = x) and
  V'(x) = x^3 - x.  CIA: E1 = dense_rhs_poly in the binomial form
   from ``cdk_moments_blocks`` (w_k = (1/N) sum_{l in c} x_l^k)
  and ``cdk_dense_poly`` with tbl[c, b] = (-1)^b sum_{a >= b} c_a C(a, b)
  w_{a-b}[c]; E2 = ``cdk_pairs_poly`` over S (exact h).  Naive: pairs_poly
  over the full edge list.
* ``rank_one_rhs`` (Appendix B.1): ``cdk_rank_one``.
* ``nearest_neighbor_rhs`` (Appendix B.2): ``cdk_nn_recurrence``
  on e^{i x}, output F_m e^{-i x_m}.
* ``BornholdtRohlf`` / ``iterate_map``: f_m = sum_l v_l
  + mu v_m + sigma r_m, v_m <- sgn(f_m) (sgn(0) = +1), the field sums from
  ``cdk_spin_field_sums``, the noise drawn on the host in fixed node order
  (PCG64(seed), N standard normals per step) and uploaded.

All state stays on the device between stages; the RK4/Euler combination of
Desai–Zwanzig stages uses device tensor arithmetic in the oracle's order
(oracle/cia.py:82-102).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from math import comb

import numpy as np

from . import _kernels, _lib
from .errors import BlowUpError, InputError
from .graph import Decomposition, Graph


def _t(a, dtype=None):
    import torch

    return torch.as_tensor(np.asarray(a, dtype=dtype) if not torch.is_tensor(a) else a,
                           device="cuda")


# ---------------------------------------------------------------------------
# Desai–Zwanzig
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class DesaiZwanzig:
    """x' = -V'(x) + (1/N) sum_l a_ml h(x_l - x_m); h(d) = sum_a coef[a] d^a."""

    n_nodes: int
    coef: np.ndarray = field(default_factory=lambda: np.array([0.0, 1.0]))
    v_prime: tuple = (0.0, -1.0, 0.0, 1.0)  # V'(x) = sum_k v_prime[k] x^k (x^3 - x)
    norm: float | None = None
    state_space: str = "real"

    def norm_value(self) -> float:
        return float(self.norm if self.norm is not None else self.n_nodes)


def _dense_table(coef: np.ndarray, w):
    """tbl[c, b] = (-1)^b sum_{a >= b} coef[a] C(a, b) w[c, a - b] (device)."""
    import torch

    p = coef.shape[0] - 1
    tbl = torch.zeros((w.shape[0], p + 1), dtype=torch.float64, device=w.device)
    for b in range(p + 1):
        acc = torch.zeros(w.shape[0], dtype=torch.float64, device=w.device)
        for a in range(b, p + 1):
            if coef[a] != 0.0:
                acc = acc + float(coef[a] * comb(a, b)) * w[:, a - b]
        tbl[:, b] = acc if b % 2 == 0 else -acc
    return tbl


class DzEngine:
    """Desai–Zwanzig right-hand side, CIA (a Decomposition, permuted order) or
    naive (a Graph, the graph's node order)."""

    def __init__(self, model: DesaiZwanzig, target):
        import torch

        _lib.lib()
        self.model = model
        self.coef = np.asarray(model.coef, dtype=np.float64)
        self.coef_t = _t(self.coef, np.float64)
        self.inv_n = 1.0 / model.norm_value()
        self.cia = isinstance(target, Decomposition)
        if self.cia:
            s = target.correction
            self.offsets = _t(target.offsets, np.int64)
            self.iu, self.iv = _t(s.iu, np.int64), _t(s.iv, np.int64)
            self.sgn = _t(s.sgn, np.float64)
            self.n = target.n_nodes
        elif isinstance(target, Graph):
            e = target.edges
            self.iu, self.iv = _t(e[:, 0].copy(), np.int64), _t(e[:, 1].copy(), np.int64)
            self.sgn = torch.ones(e.shape[0], dtype=torch.float64, device="cuda")
            self.n = target.n_nodes
        else:
            raise InputError("DzEngine needs a Decomposition (cia) or a Graph (naive)")

    def intrinsic(self, x):
        """-V'(x) by Horner (device)."""
        import torch

        vp = self.model.v_prime
        acc = torch.full_like(x, float(vp[-1]))
        for k in range(len(vp) - 2, -1, -1):
            acc = acc * x + float(vp[k])
        return -acc

    def rhs(self, x):
        import torch

        x = _t(x, np.float64).contiguous()
        out = self.intrinsic(x).contiguous()
        if self.cia:
            p = self.coef.shape[0] - 1
            w = _kernels.moments_blocks(x, self.offsets, p, 0.0, 1.0 / self.inv_n)
            tbl = _dense_table(self.coef, w)
            _kernels.dense_poly(x, self.offsets, tbl, 1.0, 0.0, out)
        _kernels.pairs_poly(self.iu, self.iv, x, self.inv_n, self.coef_t, 0.0, self.sgn, out)
        return out

    def rk4(self, x, dt: float, n_steps: int):
        import torch

        x = _t(x, np.float64).clone()
        h2, h6 = dt / 2.0, dt / 6.0
        for s in range(1, n_steps + 1):
            k1 = self.rhs(x)
            k2 = self.rhs(x + h2 * k1)
            k3 = self.rhs(x + h2 * k2)
            k4 = self.rhs(x + dt * k3)
            x = x + h6 * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
            if not bool(torch.isfinite(x).all()):
                raise BlowUpError(s)
        return x


# ---------------------------------------------------------------------------
# Appendix B fast paths
# ---------------------------------------------------------------------------
def rank_one_rhs(alpha, beta, x):
    """alpha_m r e^{-i x_m}, r = (1/N) sum_l beta_l e^{i x_l} (complex [N])."""
    import torch

    a, b, xt = _t(alpha, np.float64), _t(beta, np.float64), _t(x, np.float64)
    n = xt.shape[0]
    if a.shape != (n,) or b.shape != (n,):
        raise InputError("alpha, beta and x must have the same length")
    out = torch.empty(n, dtype=torch.complex128, device="cuda")
    scratch = torch.empty(148 * 2, dtype=torch.float64, device="cuda")
    L = _lib.lib()
    _lib.check(L.cdk_rank_one(a.data_ptr(), b.data_ptr(), xt.data_ptr(), n, 1.0 / max(n, 1),
                              out.data_ptr(), scratch.data_ptr(), _lib.stream_ptr()), "rank_one")
    return out.cpu().numpy()


def nearest_neighbor_rhs(k: int, x, anchor_every: int = 1024):
    """F_m e^{-i x_m} with F_m = (1/N) sum_{l=m-k..m+k} e^{i x_l} (ring, window
    capped at N - 1 neighbours)."""
    import torch

    xt = _t(x, np.float64)
    n = int(xt.shape[0])
    if k < 1:
        raise InputError("k >= 1")
    k = min(int(k), (n - 1) // 2) if n > 1 else 0
    ph = torch.exp(1j * xt.to(torch.complex128))
    f = _kernels.nn_recurrence(ph, k, 1.0 / n, anchor_every)
    return (f * torch.exp(-1j * xt.to(torch.complex128))).cpu().numpy()


# ---------------------------------------------------------------------------
# Bornholdt–Rohlf
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class BornholdtRohlf:
    mu: float = 1.0
    sigma: float = 0.0


def iterate_map(model: BornholdtRohlf, v0, steps: int, seed: int = 0) -> np.ndarray:
    """Synchronous spin updates; returns the states [steps + 1, N] (int8)."""
    import torch

    v = _t(np.asarray(v0, dtype=np.int64), np.int64)
    if not bool(((v == 1) | (v == -1)).all()):
        raise InputError("spins must be -1 or +1")
    rng = np.random.Generator(np.random.PCG64(seed))
    states = [v.cpu().numpy().astype(np.int8)]
    for _ in range(int(steps)):
        fs = _kernels.spin_field_sums(v)  # sum_l v_l for every m (exact int64)
        noise = rng.standard_normal(v.shape[0]) if model.sigma != 0.0 else None
        f = fs.to(torch.float64) + model.mu * v.to(torch.float64)
        if noise is not None:
            f = f + model.sigma * _t(noise, np.float64)
        v = torch.where(f >= 0.0, 1, -1).to(torch.int64)  # sgn(0) = +1
        states.append(v.cpu().numpy().astype(np.int8))
    return np.stack(states)
