"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the SPEC orchestration that the reference declares but does
not ship, composed ONLY of reference-kernel calls (``kern`` is either
``oracle.kernels`` — the C restatement — or the real reference module
``commdyn._kernels``; tests/golden/make_golden.py runs this same code on the
latter to pin the former):

* ``kuramoto_rhs_cia``    SPEC.md:359-366 (eval_rhs_cia) + :433-438 (kuramoto_rhs):
                          f = omega; E1 order_params_blocks + dense_complex;
                          E2 pairs_trig with exact sin over S
* ``kuramoto_rhs_naive``  SPEC.md:368-374: direct sum over the full edge list
                          (pairs_trig with sgn = +1, no dense part)
* ``rk4_integrate``       SPEC.md:517-536: classical RK4, phases wrapped to
                          (-pi, pi] after each full step,
                          non-finite state -> BlowUpError(step)

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import it.
"""

from __future__ import annotations

import math

import numpy as np

TWO_PI = 2.0 * math.pi


def wrap_phase(x):
    """(-pi, pi] representative.  Same formula as the CUDA path."""
    return x - TWO_PI * np.ceil((x - math.pi) / TWO_PI)


def circ_dist(a, b):
    """Circular distance between phase arrays."""
    d = np.abs(np.asarray(a) - np.asarray(b)) % TWO_PI
    return np.minimum(d, TWO_PI - d)


def kuramoto_tables(coupling: float):
    """Coefficients of h = coupling * sin on L = pi, p = 1."""
    d = {1: coupling / 2j, 0: 0.0 + 0.0j, -1: -coupling / 2j}
    d_cos = np.array([0.0, 0.0])
    d_sin = np.array([0.0, float(coupling)])
    return d, d_cos, d_sin


def kuramoto_rhs_cia(kern, theta, omega, offsets, iu, iv, sgn, coupling, norm, out=None):
    """theta' = omega + (coupling/norm) sum_l A_ml sin(theta_l - theta_m), CIA form."""
    p = 1
    d, d_cos, d_sin = kuramoto_tables(coupling)
    out = np.array(omega, dtype=np.float64, copy=True) if out is None else out
    r = kern.order_params_blocks(theta, offsets, p, math.pi, norm)
    tbl = np.zeros_like(r)
    for a in (-1, 0, 1):  # tbl[c, p - a] = d_a r[c, p + a]
        tbl[:, p - a] = d[a] * r[:, p + a]
    n_viol, max_imag = kern.dense_complex(theta, offsets, tbl, math.pi, out)
    if n_viol:
        from paper_2203_16657_b200.errors import ImagResidueError

        raise ImagResidueError(f"{n_viol} nodes above IMAG_TOL (max {max_imag:g})")
    kern.pairs_trig(iu, iv, theta, 1.0 / norm, d_cos, d_sin, math.pi, sgn, out)
    return out


def harmonics_tables(d_cos, d_sin):
    """Complex coefficients d_a (a = -p..p) of h(x) = sum_a d_cos[a] cos(a x)
    + d_sin[a] sin(a x): d_0 = d_cos[0], d_a = (d_cos[a] - i d_sin[a]) / 2,
    d_-a = conj(d_a) (SPEC.md:169-176 conversion)."""
    p = len(d_cos) - 1
    d = {0: complex(d_cos[0], 0.0)}
    for a in range(1, p + 1):
        d[a] = complex(d_cos[a], -d_sin[a]) / 2.0
        d[-a] = d[a].conjugate()
    return d


def harmonics_rhs_cia(kern, theta, omega, offsets, iu, iv, sgn, d_cos, d_sin, norm):
    """Higher-harmonics Kuramoto, CIA form over the
    reference kernels: E1 order_params_blocks (p modes) + dense_complex with
    tbl[c, p - a] = d_a r_a, E2 pairs_trig with the p harmonics (exact h)."""
    d_cos = np.asarray(d_cos, np.float64)
    d_sin = np.asarray(d_sin, np.float64)
    p = d_cos.shape[0] - 1
    d = harmonics_tables(d_cos, d_sin)
    out = np.array(omega, dtype=np.float64, copy=True)
    r = kern.order_params_blocks(theta, offsets, p, math.pi, norm)
    tbl = np.zeros_like(r)
    for a in range(-p, p + 1):
        tbl[:, p - a] = d[a] * r[:, p + a]
    n_viol, max_imag = kern.dense_complex(theta, offsets, tbl, math.pi, out)
    if n_viol:
        from paper_2203_16657_b200.errors import ImagResidueError

        raise ImagResidueError(f"{n_viol} nodes above IMAG_TOL (max {max_imag:g})")
    kern.pairs_trig(iu, iv, theta, 1.0 / norm, d_cos, d_sin, math.pi, sgn, out)
    return out


def kuramoto_rhs_naive(kern, theta, omega, eu, ev, coupling, norm):
    """Direct sum over the graph's edge list (eu < ev), exact sin."""
    _, d_cos, d_sin = kuramoto_tables(coupling)
    out = np.array(omega, dtype=np.float64, copy=True)
    kern.pairs_trig(eu, ev, theta, 1.0 / norm, d_cos, d_sin, math.pi,
                    np.ones(eu.shape[0]), out)
    return out


def kuramoto_rhs_dense(theta, omega, adj, coupling, norm):
    """Literal O(N^2) double loop in matrix form (small N only)."""
    diff = theta[None, :] - theta[:, None]
    return omega + (coupling / norm) * (adj * np.sin(diff)).sum(axis=1)


def rk4_integrate(rhs, x0, dt: float, steps: int, wrap: bool = True, record_every: int = 0):
    """Classical RK4.  Returns (final, snapshots list of (step, x))."""
    x = np.array(x0, dtype=np.float64, copy=True)
    h2 = dt / 2.0
    h6 = dt / 6.0
    snaps = []
    for step in range(1, steps + 1):
        k1 = rhs(x)
        k2 = rhs(x + h2 * k1)
        k3 = rhs(x + h2 * k2)
        k4 = rhs(x + dt * k3)
        x = x + h6 * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
        if wrap:
            x = wrap_phase(x)
        if not np.all(np.isfinite(x)):
            from paper_2203_16657_b200.errors import BlowUpError

            raise BlowUpError(step)
        if record_every and step % record_every == 0:
            snaps.append((step, x.copy()))
    return x, snaps


def euler_integrate(rhs, x0, dt: float, steps: int, wrap: bool = True):
    x = np.array(x0, dtype=np.float64, copy=True)
    for _ in range(steps):
        x = x + dt * rhs(x)
        if wrap:
            x = wrap_phase(x)
    return x
